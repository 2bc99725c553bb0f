set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
