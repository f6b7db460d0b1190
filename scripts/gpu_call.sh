python scripts/ab_lib.py paper_2511_20834_b200/libspc.so paper_2511_20834_b200/exp_notrace.so paper_2511_20834_b200/exp_notrace_nopf.so
(cd build_b9ea1a1 && python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-tune --t-from t_line.json 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('b9ea1a1', round(d['value'],1))")
python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-tune --t-from t_line.json 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('head', round(d['value'],1))"
