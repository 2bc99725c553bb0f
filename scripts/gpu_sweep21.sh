O=gpurun_out/sweep21; mkdir -p $O
for m in fma dir; do
  r=$(PE_IV_NEXT=$m timeout 600 python scripts/profile_one.py --config c5 --points 100000000 --reps 3 2>&1 | tail -1)
  echo "c5 1e8 PE_IV_NEXT=$m :: $r" >> $O/c5.txt
  PE_IV_NEXT=$m ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$m.csv \
    python scripts/profile_one.py --config c5 --points 10000000 --reps 2 > /dev/null 2>&1
done
PE_IV_NEXT=dir timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -k "interval or partition" > $O/pytest_dir.log 2>&1; echo "exit $?" >> $O/pytest_dir.log
