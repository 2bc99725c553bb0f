timeout 1500 python -m pytest tests/test_gpu_random.py -x -q -m gpu > gpurun_out/pytest_random.log 2>&1; echo "exit $?" >> gpurun_out/pytest_random.log
