timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -m gpu -k "out_of_bounds" > gpurun_out/pytest_oob.log 2>&1; echo "exit $?" >> gpurun_out/pytest_oob.log
