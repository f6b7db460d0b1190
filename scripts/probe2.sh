for lib in exp_OLD libspc exp_BOTH; do
echo $lib
for c in "128 96" "32 32" "64 64"; do set -- $c
PROBE_KERNELS=1 SPC_LIB_OVERRIDE=$PWD/paper_2511_20834_b200/$lib.so python scripts/probe_conv.py --cin $1 --cout $2 --t -1 --reps 30 2>&1 | grep -v Warn | tail -1
done; done
for n in 45000 18000 6000; do for c in 32 64 128; do
echo "n=$n c=$c  auto / bm128-template / ws"
python scripts/probe_conv.py --n $n --cin $c --cout $c --t -1 --reps 30
SPC_BM128=1 python scripts/probe_conv.py --n $n --cin $c --cout $c --t -1 --reps 30
python scripts/probe_conv.py --n $n --cin $c --cout $c --t 0 --reps 30
done; done
