timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 100 --warmup 5 --no-cpu-baseline --t-from profiles/r2_tuned_t_c2.json > gpurun_out/r2_bench_e.json 2> gpurun_out/r2_bench_e.err
python -c "import json;d=json.loads(open('gpurun_out/r2_bench_e.json').read().splitlines()[-1]);print(d['value'],d['e2e']['value']);[print(l['name'],l['us']) for l in d['layers'] if l['c_out']>=192]"
python scripts/probe_conv.py --opt CONV_CTA_PAIR=0 --cin 256 --cout 256 --t 0 --reps 10 --config 2 --n 2700 2>&1 | grep n=
python scripts/probe_conv.py --opt CONV_CTA_PAIR=1 --cin 256 --cout 256 --t 0 --reps 10 --config 2 --n 2700 2>&1 | grep n=
