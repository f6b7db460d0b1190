python scripts/timeline.py --out gpurun_out/r2_timeline4.json > gpurun_out/r2_timeline4.txt 2>&1; tail -3 gpurun_out/r2_timeline4.txt
python bench.py --steps 100 --warmup 5 --no-cpu-baseline --t-from profiles/r2_tuned_t_c2.json --profile-layers > gpurun_out/r2_bench_i.json 2> gpurun_out/r2_bench_i.err
python -c "import json;d=json.loads(open('gpurun_out/r2_bench_i.json').read().splitlines()[-1]);print(d['value'],d['e2e']['value'],d['roofline']['frac'],d['roofline']['conv_ms_per_step'],d['roofline']['index_ms_per_step'])"
