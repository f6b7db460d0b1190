#!/bin/bash
# Round-2 ncu evidence for the current build (run under gpurun from the repo root; 1 GPU).
# Summaries land in gpurun_out/ (copy the ones to keep into profiles/).
set -x
T=${T_FROM:-profiles/r2_tuned_t_c2.json}
O=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $O/r2_launches.csv python scripts/one_pass.py --t-from $T > $O/r2_launches.log 2>&1
python scripts/summarize_ncu.py launches $O/r2_launches.csv $O/r2_launches.md
timeout 1500 ncu --set full --clock-control none --profile-from-start off -k regex:"k_conv_tc|k_convert|k_dense_tc" \
  -o $O/r2_conv_all -f python scripts/one_pass.py --t-from $T > $O/r2_conv_all.log 2>&1
python scripts/conv_traffic.py $O/r2_conv_all.ncu-rep $O/r2_conv_traffic_c2.json --config 2 --n-voxels 98895
python scripts/summarize_ncu.py full $O/r2_conv_all.ncu-rep $O/r2_conv_full.txt
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_kmap_zdelta|k_onesweep|k_ord_permute|k_kmap_bounds" -c 8 -o $O/r2_index_full -f python scripts/one_pass.py --t-from $T > $O/r2_index_full.log 2>&1
python scripts/summarize_ncu.py full $O/r2_index_full.ncu-rep $O/r2_index_full.txt
for cfg in "256 256 -1 0" "256 256 -1 1" "128 128 -1 -1" "192 192 -1 1" "256 256 2 -1" "96 96 -1 -1"; do
  set -- $cfg
  timeout 300 ncu --set full --clock-control none -k regex:k_conv_tc -s 2 -c 1 -o $O/r2_wide_$1_$2_t$3_p$4 -f \
    python scripts/probe_conv.py --cin $1 --cout $2 --t $3 --pair $4 --reps 1 --config 5 > /dev/null 2>&1
  python scripts/summarize_ncu.py full $O/r2_wide_$1_$2_t$3_p$4.ncu-rep $O/r2_wide_$1_$2_t$3_p$4.txt
  timeout 120 python scripts/probe_conv.py --cin $1 --cout $2 --t $3 --pair $4 --reps 20 --config 5 >> $O/r2_wide_times.log 2>&1
done
timeout 1500 python scripts/sweep_c5.py $O/r2_c5_sweep.md > $O/r2_c5_sweep.jsonl 2> $O/r2_c5_sweep.err
rm -f $O/r2_conv_all.ncu-rep $O/r2_index_full.ncu-rep
ls -la $O
