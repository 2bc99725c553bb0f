timeout 2400 bash scripts/gpu_sweep7.sh > gpurun_out/sweep7.log 2>&1
