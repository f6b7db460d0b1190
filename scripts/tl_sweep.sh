for n in 8000 20000 45000; do
  for c in "32 32" "64 64" "128 128"; do
    set -- $c
    echo "== n=$n cin=$1 cout=$2 t=-1"
    SPC_LIB_OVERRIDE=$PWD/paper_2511_20834_b200/exp_TL.so timeout 60 python scripts/timeline_conv.py --cin $1 --cout $2 --t -1 --n $n 2>&1 | tail -9
  done
done
