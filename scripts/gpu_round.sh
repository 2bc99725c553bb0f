timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu -k "interval or deferred" > gpurun_out/pytest_iv.log 2>&1; echo "exit $?" >> gpurun_out/pytest_iv.log
for m in hybrid fma; do PE_IV_NEXT=$m timeout 300 python scripts/profile_one.py --config c5 --reps 3 2>&1 | tail -1 | sed "s/^/$m /"; done > gpurun_out/c5_next.log 2>&1
