set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest.log
for c in c4 c3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
for K in 1 2 3 4 6 8; do PE_SLICES=$K timeout 600 python scripts/profile_one.py --config c4 --points 4000000 --reps 3 2>&1 | tail -1 | sed "s/^/K=$K /"; done > gpurun_out/slices_c4.log 2>&1
