#!/bin/bash
# Round-2 (second session) evidence for the final build: GPU parity, smoke, bench lines,
# training step, wgrad probe + ncu, C2 launch list, C5 sweep.  Run under gpurun from the
# repo root (1 GPU); summaries land in gpurun_out/ (copy the ones to keep into profiles/).
set -x
O=gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > $O/gputest_final.log 2>&1; echo "rc=$?" >> $O/gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_final.log 2>&1
timeout 400 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --config 1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 400 python bench.py --config 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config 4 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 400 python bench.py --net minkunet42_k2 > $O/bench_c2_k2.json 2> $O/bench_c2_k2.err
timeout 300 python scripts/train_bench.py > $O/train_c2.json 2> $O/train_c2.err
for cfg in "0 32 32" "0 96 96" "1 128 96" "2 128 128" "3 256 256" "4 256 256"; do
  set -- $cfg
  timeout 120 python scripts/probe_wgrad.py --level $1 --cin $2 --cout $3 >> $O/wgrad_probe.log 2>&1
done
timeout 300 python scripts/index_phases.py > $O/index_phases.log 2>&1
timeout 300 python scripts/index_phases.py --config 4 >> $O/index_phases.log 2>&1
T=profiles/r2_tuned_t_c2.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $O/r2b_launches.csv python scripts/one_pass.py --t-from $T > $O/r2b_launches.log 2>&1
python scripts/summarize_ncu.py launches $O/r2b_launches.csv $O/r2b_launches.md
for cfg in "0 96 96" "3 256 256"; do
  set -- $cfg
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_wgrad_tc -s 1 -c 1 -o $O/wgrad_$1_$2 -f \
    python scripts/probe_wgrad.py --level $1 --cin $2 --cout $3 --reps 2 > /dev/null 2>&1
  python scripts/summarize_ncu.py full $O/wgrad_$1_$2.ncu-rep $O/r2_wgrad_full_l$1_$2.txt
  rm -f $O/wgrad_$1_$2.ncu-rep
done
timeout 2000 python scripts/sweep_c5.py $O/r2_c5_sweep.md > $O/r2_c5_sweep.jsonl 2> $O/r2_c5_sweep.err
ls -la $O
