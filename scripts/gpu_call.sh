set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --steps 50 --warmup 5 --profile-layers --no-cpu-baseline > gpurun_out/r2_base_bench.json 2> gpurun_out/r2_base_layers.txt
tail -c 3000 gpurun_out/r2_base_bench.json
