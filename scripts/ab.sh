#!/bin/bash
# A/B env settings on the C2 bench (run under gpurun)
O=gpurun_out
for envs in "" "SPC_NO_FUSED_CVT=1" "SPC_SPLIT_TILES2=1024" "SPC_SPLIT_TILES2=600" "SPC_SPLIT_TILES2=1024 SPC_SPLIT_MIN=4"; do
  env $envs timeout 300 python bench.py --steps 100 --t-from profiles/r1_bench.json --no-cpu-baseline > $O/ab.json 2> $O/ab.err
  python -c "import json;d=json.load(open('$O/ab.json'));print('[$envs]', round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['conv_ms_per_step'],4))"
done
