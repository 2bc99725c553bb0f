timeout 2400 python scripts/setup_bench.py > gpurun_out/setup_bench.log 2>&1; echo "exit $?" >> gpurun_out/setup_bench.log
