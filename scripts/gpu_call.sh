set -x
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" 
python bench.py --config 1 --steps 200 --warmup 5 > gpurun_out/r2_bench_c1.json 2> gpurun_out/r2_bench_c1.err; tail -c 600 gpurun_out/r2_bench_c1.json; tail -3 gpurun_out/r2_bench_c1.err
python bench.py --steps 100 --warmup 5 --t-from profiles/r2_tuned_t_c2.json > gpurun_out/r2_bench_d.json 2> gpurun_out/r2_bench_d.err; tail -3 gpurun_out/r2_bench_d.err
python -c "import json;d=json.loads(open('gpurun_out/r2_bench_d.json').read().splitlines()[-1]);print(d['value'],d['cpu_baseline'],d['kmap'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; tail -c 800 gpurun_out/r2_ref.json; tail -3 gpurun_out/r2_ref.err
