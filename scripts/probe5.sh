for lib in exp_TL; do
export SPC_LIB_OVERRIDE=$PWD/paper_2511_20834_b200/$lib.so
for cfg in "18000 128 128"; do set -- $cfg
echo "== $lib n=$1 cin=$2 cout=$3"
python scripts/timeline_conv.py --n $1 --cin $2 --cout $3 --t -1 2>&1 | grep -E "last_commit|exit|last |end "
done; done
