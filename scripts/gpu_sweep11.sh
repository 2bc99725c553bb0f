# C5: finite-case replay in the fixup entry (PE_IV_MID=1, default) vs the
# bit-level replay only (PE_IV_MID=0); interval parity tests.
O=gpurun_out/sweep11; mkdir -p $O
{
for m in 0 1; do
  r=$(PE_IV_MID=$m timeout 600 python scripts/profile_one.py --config c5 --points 10000000 --reps 4 2>&1 | tail -1)
  echo "c5 1e7 PE_IV_MID=$m :: $r"
  r=$(PE_IV_MID=$m timeout 600 python scripts/profile_one.py --config c5 --points 100000000 --reps 3 2>&1 | tail -1)
  echo "c5 1e8 PE_IV_MID=$m :: $r"
done
} > $O/c5.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "interval or edges or random or parity" > $O/pytest_iv.log 2>&1; echo "exit $?" >> $O/pytest_iv.log
nsys_dummy=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
    python scripts/profile_one.py --config c5 --points 10000000 --reps 3 > /dev/null 2>&1
