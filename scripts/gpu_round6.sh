#!/bin/bash
# Final round-1 bench set (steps enqueued back to back inside the bracket).
O=gpurun_out/round6; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference > $O/bench_reference_c2.json 2> $O/bench_reference_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
  python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
echo done > $O/DONE
