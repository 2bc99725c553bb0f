# C5 fixup entry occupancy (.minnctapersm via PE_FIX_CTAS) with the
# finite-case replay; classifier with all loads in flight.
O=gpurun_out/sweep16; mkdir -p $O
for c in 4 6 8; do
  r=$(PE_FIX_CTAS=$c timeout 600 python scripts/profile_one.py --config c5 --points 100000000 --reps 3 2>&1 | tail -1)
  echo "c5 1e8 FIX_CTAS=$c :: $r" >> $O/c5.txt
  PE_FIX_CTAS=$c ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_fix$c.csv \
    python scripts/profile_one.py --config c5 --points 100000000 --reps 2 > /dev/null 2>&1
done
