set -x
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/pytest_full.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --leak-check none python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/memcheck.log 2>&1; echo "memcheck exit $?" >> gpurun_out/memcheck.log
