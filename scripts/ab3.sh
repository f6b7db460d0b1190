O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "conv or network" 2>&1 | tail -1
for envs in "SPC_CLAIM_AHEAD=1" "SPC_CLAIM_AHEAD=2" "SPC_CLAIM_AHEAD=3"; do
  env $envs timeout 300 python bench.py --steps 100 --t-from profiles/r1_bench.json --no-cpu-baseline > $O/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('$O/ab.json'));print('[$envs] C2', round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['conv_ms_per_step'],4))"
done
