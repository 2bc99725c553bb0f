# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s33; mkdir -p $O
timeout 400 python scripts/fuzz_wide.py 300 800000 > $O/fuzz_wide.json 2>$O/fuzz_wide.err
