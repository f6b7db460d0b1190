#!/bin/bash
# quick GPU check: parity tests, C4 kernel-map build timing, C2 bench (run under gpurun)
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/q_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/q_tests.log
timeout 300 python scripts/kmap_c4.py > $O/q_kmap_c4.json 2> $O/q_kmap_c4.err; python -c "import json;d=json.load(open('$O/q_kmap_c4.json'));print('kmap_c4', d['median_us'], d['achieved_gbs'], d['frac'])"
timeout 300 python scripts/kmap_c4.py --no-order > $O/q_kmap_c4_noord.json 2>> $O/q_kmap_c4.err; python -c "import json;d=json.load(open('$O/q_kmap_c4_noord.json'));print('kmap_c4 no-order', d['median_us'], d['achieved_gbs'], d['frac'])"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none \
  --csv --log-file $O/q_kmap_c4_ncu.csv python scripts/kmap_c4.py --reps 1 > /dev/null 2>&1
timeout 400 python bench.py --steps 100 --t-from profiles/r1_bench.json --no-cpu-baseline > $O/q_bench.json 2> $O/q_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/q_bench.json'));print('bench', d['value'], d['ms_per_step'], d['roofline']['conv_ms_per_step'], d['roofline']['index_ms_per_step'], d['e2e']['value'])"
if [ -n "$LAUNCHES" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $O/q_launches.csv python scripts/one_pass.py --t-from profiles/r1_bench.json > $O/q_launches.log 2>&1
  python scripts/summarize_ncu.py launches $O/q_launches.csv $O/q_launches.md
  head -16 $O/q_launches.md
fi
