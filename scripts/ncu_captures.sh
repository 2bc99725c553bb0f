#!/bin/bash
# Launch lists and `ncu --set full` captures of the bench's dominant kernels at
# the bench's own launch sizes (one GPU; each command first runs clean
# without ncu). Outputs under gpurun_out/ncu/; copy the summaries to profiles/.
#   bash scripts/ncu_captures.sh [c4] [c5] ...
O=gpurun_out/ncu; mkdir -p $O
for c in "${@:-c4 c5}"; do
  cfg=$c; tune=""
  case $c in
    c4) pts=100000000; k="regex:pe_walk" ;;
    c5) pts=100000000; k="regex:pe_walk|classify" ;;
    c5split) pts=100000000; k="regex:pe_walk"; cfg=c5; tune="--tune jit_mode=1,iv_partition=3" ;;
    *) pts=10000000; k="regex:pe_walk" ;;
  esac
  python scripts/profile_one.py --config $cfg --points $pts --reps 1 $tune > $O/${c}_plain.log 2>&1 || continue
  [ -z "$tune" ] && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${c}.csv \
    python bench.py --config ${c:0:2} --steps 2 --warmup 3 --no-cpu --no-e2e > $O/${c}_launches.log 2>&1
  ncu --set full --import-source on --clock-control none -k $k -s 1 -c 4 \
    -o $O/ncu_${c} python scripts/profile_one.py --config $cfg --points $pts --reps 1 $tune > $O/${c}_ncu.log 2>&1
  ncu -i $O/ncu_${c}.ncu-rep --page raw --csv > $O/r2_ncu_${c}_raw.csv 2>/dev/null
  ncu -i $O/ncu_${c}.ncu-rep --page details --csv > $O/r2_ncu_${c}_details.csv 2>/dev/null
  echo $pts > $O/r2_ncu_${c}_points.txt
  rm -f $O/ncu_${c}.ncu-rep  # gpurun copies back at most 64 MiB: keep the CSV exports only
done
echo done > $O/DONE
