for envs in "" "SPC_BM256_SINGLE=1" "SPC_BM256_SINGLE=1 SPC_STAGE_KB=128"; do
  env $envs PROBE_KERNELS=1 timeout 120 python scripts/probe_conv.py --cin 256 --cout 256 --t -1 --reps 20 2>&1 | grep -v Warn | head -3 | sed "s/^/[$envs] /"
done
