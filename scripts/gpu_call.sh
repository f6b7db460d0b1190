set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --steps 100 --warmup 5 --no-cpu-baseline --t-from profiles/r2_tuned_t_c2.json --profile-layers > gpurun_out/r2_bench_b.json 2> gpurun_out/r2_bench_b.err
tail -c 1200 gpurun_out/r2_bench_b.json
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_c1.py --small > gpurun_out/r2_sanitize_racecheck.txt 2>&1; echo "racecheck rc=$?"
tail -3 gpurun_out/r2_sanitize_racecheck.txt
