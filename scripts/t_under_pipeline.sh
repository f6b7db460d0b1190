O=gpurun_out/tprobe.log
run() { timeout 300 python scripts/pipeline_probe.py --afters 19 --splitsets 22 "$@" 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['sequential_ms'],4), round(d['ms_cap0_prio0_after19'],4), round(d['ms_split22'],4))" >> $O; }
run
run --t-set 3,1,8,0=4 --t-set 3,1,16,0=4
run --t-set 3,1,8,0=2 --t-set 3,1,16,0=2
run --t-set 3,2,4,0=4 --t-set 3,2,8,0=4 --t-set 3,2,8,1=4
run --t-set 3,1,4,0=2
run --t-set 3,1,1,0=3 --t-set 3,1,2,0=3
