#!/bin/bash
# Round-1 re-measurement after the coefficient-delivery change: GPU tests,
# bench c1-c5, launch lists, ncu --set full of C2 / C3 / C4.
O=gpurun_out/round2; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for c in c2 c3 c4 c5 c1; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
for c in c2 c3 c4; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:pe_walk -s 4 -c 4 \
  -o $O/ncu_c2_all python scripts/profile_c2_all.py --reps 2 > $O/ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:pe_walk -s 1 -c 1 \
  -o $O/ncu_c3 python scripts/profile_one.py --config c3 --points 10000000 --reps 2 > $O/ncu_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:pe_walk -s 4 -c 4 \
  -o $O/ncu_c4 python scripts/profile_one.py --config c4 --points 100000000 --reps 2 > $O/ncu_c4.log 2>&1
echo done > $O/DONE
