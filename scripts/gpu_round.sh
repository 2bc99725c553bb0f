set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest.log
timeout 2000 bash scripts/gpu_sweep4.sh > gpurun_out/sweep4.log 2>&1
