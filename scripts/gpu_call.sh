python scripts/indexing_modes.py --config 2 --reps 20 | tee gpurun_out/r2_indexing_modes.jsonl
python scripts/indexing_modes.py --config 4 --reps 10 | tee -a gpurun_out/r2_indexing_modes.jsonl
