timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pair.py tests/test_gpu_headline.py -q -x 2>&1 | tail -1
python scripts/ab_net.py CONV_BULK_RED=0 CONV_BULK_RED=1 2>&1 | tail -2
for o in 0 1; do python scripts/probe_conv.py --opt CONV_BULK_RED=$o --cin 256 --cout 256 --t 0 --reps 10 --config 5 2>&1 | grep "n="; python scripts/probe_conv.py --opt CONV_BULK_RED=$o --cin 256 --cout 256 --t 0 --reps 10 --config 2 --n 7000 2>&1 | grep "n="; done
