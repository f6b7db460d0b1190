for lib in exp_OLD exp_BOTH; do
SPC_LIB_OVERRIDE=$PWD/paper_2511_20834_b200/$lib.so timeout -s KILL 300 ncu --set full --clock-control none -k regex:k_conv_tc -s 2 -c 1 -o gpurun_out/ncu_$lib python scripts/probe_conv.py --cin 128 --cout 96 --t -1 --reps 1 > gpurun_out/ncu_$lib.log 2>&1
done
