# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s7; mkdir -p $O
timeout 500 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 3000 python -m pytest tests -m gpu -q --timeout 600 --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
