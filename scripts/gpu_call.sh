timeout 900 python -m pytest tests/test_gpu_keys32.py -x -q 2>&1 | tail -4
python scripts/keys32_ablation.py | tee gpurun_out/r2_keys32.jsonl
