# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s23; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 2400 python scripts/fig1_grid.py > $O/fig1_grid.jsonl 2> $O/fig1.err
