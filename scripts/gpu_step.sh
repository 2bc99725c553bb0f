# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s31; mkdir -p $O
timeout 600 python scripts/fuzz_repro.py 410119 > $O/repro_410119.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "interval or partition" > $O/pytest_iv.log 2>&1; echo "pytest exit $?" >> $O/pytest_iv.log
timeout 300 python scripts/profile_one.py --config c5 --points 100000000 --reps 3 --tune jit_mode=1 --tune jit_mode=1,iv_partition=-1 > $O/c5.jsonl 2> $O/c5.err
