set -x
python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
python scripts/timeline.py --out gpurun_out/r2_timeline2.json > gpurun_out/r2_timeline2.txt 2>&1
tail -3 gpurun_out/r2_timeline2.txt
python bench.py --steps 100 --warmup 5 --no-cpu-baseline --t-from profiles/r2_tuned_t_c2.json > gpurun_out/r2_bench_c.json 2> gpurun_out/r2_bench_c.err
head -c 400 gpurun_out/r2_bench_c.json
