O=gpurun_out/sweep19; mkdir -p $O
for o in 0 1; do
  PE_IV_OUTFMA=$o timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -k "interval or partition" > $O/pytest_out$o.log 2>&1; echo "exit $?" >> $O/pytest_out$o.log
  r=$(PE_IV_OUTFMA=$o timeout 600 python scripts/profile_one.py --config c5 --points 100000000 --reps 3 2>&1 | tail -1)
  echo "c5 1e8 OUTFMA=$o :: $r" >> $O/c5.txt
  r=$(PE_IV_OUTFMA=$o timeout 600 python scripts/profile_one.py --config c5 --points 10000000 --reps 4 2>&1 | tail -1)
  echo "c5 1e7 OUTFMA=$o :: $r" >> $O/c5.txt
done
