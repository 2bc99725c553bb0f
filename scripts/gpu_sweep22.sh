# Latency-aware reordering of fused streams (PE_SCHED="W,D").
O=gpurun_out/sweep22; mkdir -p $O
for sch in none 16,4 32,6 64,8 32,12; do
  if [ $sch = none ]; then unset PE_SCHED; else export PE_SCHED=$sch; fi
  r=$(timeout 600 python scripts/profile_one.py --config c4 --points 4000000 --reps 4 2>&1 | tail -1)
  echo "c4 SCHED=$sch :: $r" >> $O/sched.txt
  for c in c2e1000 c2b1000 c3; do
    r=$(timeout 600 python scripts/profile_one.py --config $c --points 10000000 --reps 4 2>&1 | tail -1)
    echo "$c SCHED=$sch :: $r" >> $O/sched.txt
  done
done
