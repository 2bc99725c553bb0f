timeout 1500 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pytest.log
