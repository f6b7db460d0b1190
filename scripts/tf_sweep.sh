for n in 8000 45000; do
  for c in "32 32" "128 128"; do
    set -- $c
    echo "== n=$n cin=$1 cout=$2 t=-1"
    SPC_LIB_OVERRIDE=$PWD/paper_2511_20834_b200/exp_TF.so timeout 60 python scripts/timeline_first.py --cin $1 --cout $2 --t -1 --n $n 2>&1 | tail -8
  done
done
