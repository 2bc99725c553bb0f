#!/bin/bash
# Full measurement round on the GPU box (run through gpurun from the repo
# root): smoke, GPU tests, bench per config, reference arm, ncu launch lists
# and full captures. Outputs under gpurun_out/round/.
O=gpurun_out/round
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference > $O/bench_reference_c2.json 2> $O/bench_reference_c2.err
# launch lists (same commands, cold-cache serialised per-launch times)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
for c in c1 c3 c4 c5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
# full captures of the dominant kernels
ncu --set full --import-source on --clock-control none -k regex:pe_walk -s 4 -c 4 \
  -o $O/ncu_c2_all python scripts/profile_c2_all.py --reps 2 > $O/ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:pe_walk_interval$ -s 1 -c 1 \
  -o $O/ncu_c5 python scripts/profile_one.py --config c5 --points 10000000 --reps 2 > $O/ncu_c5.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:pe_walk -s 1 -c 1 \
  -o $O/ncu_c3 python scripts/profile_one.py --config c3 --points 10000000 --reps 2 > $O/ncu_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:pe_walk -s 6 -c 6 \
  -o $O/ncu_c4 python scripts/profile_one.py --config c4 --points 4000000 --reps 2 > $O/ncu_c4.log 2>&1
echo done > $O/DONE
