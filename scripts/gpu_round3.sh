#!/bin/bash
# Final round-1 measurement set: smoke, GPU tests, bench c1-c5 + reference
# arm, launch lists, ncu --set full of C1 and the C5 partitioned call.
O=gpurun_out/round3; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference > $O/bench_reference_c2.json 2> $O/bench_reference_c2.err
for c in c1 c5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:"classify|pe_walk" -s 4 -c 4 \
  -o $O/ncu_c5 python scripts/profile_one.py --config c5 --points 100000000 --reps 2 > $O/ncu_c5.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:pe_walk -s 1 -c 1 \
  -o $O/ncu_c1 python scripts/profile_one.py --config c1 --points 100000 --reps 2 > $O/ncu_c1.log 2>&1
echo done > $O/DONE
