#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/q_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/q_tests.log
for envs in "" "SPC_NO_BM256_SINGLE=1"; do
  for c in "256 256 -1" "256 256 2" "256 256 0"; do set -- $c
    env $envs timeout 120 python scripts/probe_conv.py --cin $1 --cout $2 --t $3 --reps 20 2>&1 | tail -1 | sed "s/^/[$envs] /"
  done
done
for envs in "" "SPC_NO_BM256_SINGLE=1"; do
  env $envs timeout 300 python bench.py --steps 100 --t-from profiles/r1_bench.json --no-cpu-baseline > $O/ab.json 2> $O/ab.err
  python -c "import json;d=json.load(open('$O/ab.json'));print('[$envs] C2', round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['conv_ms_per_step'],4), round(d['roofline']['index_ms_per_step'],4))"
done
timeout 400 python bench.py --config 4 --steps 20 --no-cpu-baseline > $O/ab4.json 2> $O/ab4.err; python -c "import json;d=json.load(open('$O/ab4.json'));print('C4', round(d['value'],1), round(d['ms_per_step'],3), d['roofline']['frac'])"
timeout 300 python scripts/ablation_mapstep.py > $O/ablation_mapstep.jsonl 2> $O/ablation_mapstep.err; cat $O/ablation_mapstep.jsonl
