O=gpurun_out/sweep27; mkdir -p $O
for shape in 1,512,32 2,256,16 2,512,32 2,256,0; do
  IFS=, read L B S <<< "$shape"
  r=$(PE_LANES=$L PE_BLOCK=$B PE_SYNC=$S timeout 600 python scripts/profile_one.py --config c5 --points 100000000 --reps 3 2>&1 | tail -1)
  echo "c5 1e8 L=$L B=$B S=$S :: $r" >> $O/c5.txt
done
PE_LANES=2 PE_BLOCK=256 PE_SYNC=16 timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -k "partition" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
