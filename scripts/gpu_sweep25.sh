O=gpurun_out/sweep25; mkdir -p $O
for o in 1 2 3 4; do
  r=$(PE_IV_OUTFMA=$o timeout 600 python scripts/profile_one.py --config c5 --points 100000000 --reps 3 2>&1 | tail -1)
  echo "c5 1e8 OUTFMA=$o :: $r" >> $O/c5.txt
done
PE_IV_OUTFMA=2 timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -k "interval or partition" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
