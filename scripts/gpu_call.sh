for s in 0.0 0.5 0.8; do ./scripts/gather4_bench.bin $s; done
