#!/bin/bash
# ncu evidence for the current build (run under gpurun from the repo root; 1 GPU).
# Everything is summarised to text on the box (gpurun copies back <= 64 MiB):
# launch list of one bench pass, --set full of a few conv launches and of the kernel-map
# build, C4 kernel-map build timing + DRAM counters, wide-layer tensor-pipe captures.
set -x
T=${T_FROM:-profiles/r1_bench.json}
O=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches.csv python scripts/one_pass.py --t-from $T > $O/launches.log 2>&1
python scripts/summarize_ncu.py launches $O/launches.csv $O/launches.md
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_conv_tc" -s 30 -c 6 -o $O/conv_full -f python scripts/one_pass.py --t-from $T > $O/conv_full.log 2>&1
python scripts/summarize_ncu.py full $O/conv_full.ncu-rep $O/conv_full.txt
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_kmap_zdelta|k_onesweep|k_ord_permute" -c 6 -o $O/index_full -f python scripts/one_pass.py --t-from $T > $O/index_full.log 2>&1
python scripts/summarize_ncu.py full $O/index_full.ncu-rep $O/index_full.txt
timeout 300 python scripts/kmap_c4.py > $O/kmap_c4.json 2> $O/kmap_c4.err
timeout 300 python scripts/kmap_c4.py --t os > $O/kmap_c4_os.json 2>> $O/kmap_c4.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none \
  --csv --log-file $O/kmap_c4_ncu.csv python scripts/kmap_c4.py --reps 1 > $O/kmap_c4_ncu.log 2>&1
python scripts/ncu_table.py $O/kmap_c4_ncu.csv --last 30 > $O/kmap_c4_ncu.txt
for cfg in "256 256 -1" "256 256 2" "128 128 -1" "128 128 2"; do
  set -- $cfg
  timeout 300 ncu --set full --clock-control none -k regex:k_conv_tc -s 2 -c 2 -o $O/wide_$1_$2_t$3 -f \
    python scripts/probe_conv.py --cin $1 --cout $2 --t $3 --reps 1 > $O/wide_$1_$2_t$3.log 2>&1
  python scripts/summarize_ncu.py full $O/wide_$1_$2_t$3.ncu-rep $O/wide_$1_$2_t$3.txt
  timeout 120 python scripts/probe_conv.py --cin $1 --cout $2 --t $3 --reps 20 >> $O/wide_times.log 2>&1
done
rm -f $O/*.ncu-rep
ls -la $O
