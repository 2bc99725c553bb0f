O=gpurun_out/sweep23; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -k "c4 or slice or wide or fullsize or from_compiled or random" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for sch in 64,8 96,8 128,8 128,12 64,6; do
  r=$(PE_SCHED=$sch timeout 600 python scripts/profile_one.py --config c4 --points 4000000 --reps 4 2>&1 | tail -1)
  echo "c4 SCHED=$sch :: $r" >> $O/sched.txt
done
for k in 3 5 6; do
  r=$(PE_SLICES=$k timeout 600 python scripts/profile_one.py --config c4 --points 4000000 --reps 4 2>&1 | tail -1)
  echo "c4 SCHED=64,8 K=$k :: $r" >> $O/sched.txt
done
timeout 900 python bench.py --config c4 > $O/bench_c4.json 2> $O/bench_c4.err
