#!/bin/bash
# ncu evidence for the current build (run under gpurun from the repo root; 1 GPU).
# Outputs under gpurun_out/: launch list of one bench pass, --set full of one whole
# forward pass (conv + indexing kernels), C4 kernel-map build timing + DRAM counters,
# wide-layer tensor-pipe captures.
set -x
T=${T_FROM:-profiles/r1_bench.json}
O=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches.csv python scripts/one_pass.py --t-from $T > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_conv_tc|k_kmap|k_onesweep|k_convert" -o $O/pass_full -f python scripts/one_pass.py --t-from $T > $O/pass_full.log 2>&1
timeout 300 python scripts/kmap_c4.py > $O/kmap_c4.json 2> $O/kmap_c4.err
timeout 300 python scripts/kmap_c4.py --t os > $O/kmap_c4_os.json 2>> $O/kmap_c4.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none \
  --csv --log-file $O/kmap_c4_ncu.csv python scripts/kmap_c4.py --reps 1 > $O/kmap_c4_ncu.log 2>&1
for cfg in "256 256 -1" "256 256 2" "128 128 -1" "128 128 2"; do
  set -- $cfg
  timeout 300 ncu --set full --clock-control none -k regex:k_conv_tc -s 2 -c 2 -o $O/wide_$1_$2_t$3 -f \
    python scripts/probe_conv.py --cin $1 --cout $2 --t $3 --reps 1 > $O/wide_$1_$2_t$3.log 2>&1
  timeout 120 python scripts/probe_conv.py --cin $1 --cout $2 --t $3 --reps 20 >> $O/wide_times.log 2>&1
done
ls -la $O
