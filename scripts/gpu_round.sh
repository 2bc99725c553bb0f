# Round measurement: smoke, tests, bench (all configs), reference arm, launch list, ncu captures.
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest.log
python scripts/pcie_bw.py > gpurun_out/pcie.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks.csv 2>&1 &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 exit $?" >> gpurun_out/bench_c2.err
for c in c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c exit $?" >> gpurun_out/bench_$c.err
done
kill $SMI
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
python scripts/profile_one.py --config c2e1000 --reps 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pe_walk -s 1 -c 1 -o gpurun_out/prof_c2e_r1 python scripts/profile_one.py --config c2e1000 --reps 2 > gpurun_out/ncu_full.log 2>&1
python scripts/profile_one.py --config c5 --reps 3 > gpurun_out/prof_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pe_walk_interval$ -s 1 -c 1 -o gpurun_out/prof_c5_r1 python scripts/profile_one.py --config c5 --reps 2 > gpurun_out/ncu_c5.log 2>&1
echo done
