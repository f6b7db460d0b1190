export SPC_LIB_OVERRIDE=$PWD/paper_2511_20834_b200/exp_TL.so
for cfg in "18000 64 64" "18000 128 128" "6000 128 128" "45000 32 32" "0 128 96"; do set -- $cfg
echo "== n=$1 cin=$2 cout=$3"
python scripts/timeline_conv.py --n $1 --cin $2 --cout $3 --t -1 2>&1 | grep -v Warn
done
