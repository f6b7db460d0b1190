set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -25
python bench.py --steps 100 --warmup 5 --no-cpu-baseline --save-t profiles/r2_tuned_t_c2.json > gpurun_out/r2_bench_a.json 2> gpurun_out/r2_bench_a.err
tail -c 1500 gpurun_out/r2_bench_a.json
cp profiles/r2_tuned_t_c2.json gpurun_out/ 2>/dev/null
python -m pytest tests/test_gpu_headline.py -q -x 2>&1 | tail -5
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_c1.py > gpurun_out/r2_sanitize_$tool.txt 2>&1; echo "$tool rc=$?"
  tail -3 gpurun_out/r2_sanitize_$tool.txt
done
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_c1.py --small > gpurun_out/r2_sanitize_racecheck.txt 2>&1; echo "racecheck rc=$?"
tail -3 gpurun_out/r2_sanitize_racecheck.txt
