timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pair.py -q -x 2>&1 | tail -1
python scripts/ab_lib.py paper_2511_20834_b200/exp_prev.so paper_2511_20834_b200/libspc.so
