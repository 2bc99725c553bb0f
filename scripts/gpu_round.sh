set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest.log
timeout 1200 bash scripts/gpu_sweep5.sh > gpurun_out/sweep5.log 2>&1
