O=gpurun_out/wide_sweep.log
for pair in 0 1; do
 for skb in 48 72 96 128; do
  for ca in 1 2; do
   timeout 60 python scripts/probe_conv.py --cin 256 --cout 256 --t -1 --config 5 --reps 20 --pair $pair --opt CONV_STAGE_KB=$skb --opt CONV_CLAIM_AHEAD=$ca 2>&1 | tail -1 | sed "s/^/pair=$pair skb=$skb ca=$ca /" >> $O
  done
 done
done
for skb in 48 72 96 128; do
  timeout 60 python scripts/probe_conv.py --cin 128 --cout 128 --t -1 --config 5 --reps 20 --opt CONV_STAGE_KB=$skb 2>&1 | tail -1 | sed "s/^/128 skb=$skb /" >> $O
done
