O=gpurun_out/sweep18; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -k "small or chain" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
{
for m in 0 1048576; do
  r=$(PE_SMALL_MAX=$m timeout 600 python bench.py --config c1 --no-cpu --no-e2e --steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "c1 1e5 SMALL_MAX=$m :: ms_per_step frac $r"
  for n in 1000000 4000000; do
    r=$(PE_SMALL_MAX=$m timeout 600 python scripts/profile_one.py --config c1 --points $n --reps 4 2>&1 | tail -1)
    echo "c1 n=$n SMALL_MAX=$m :: $r"
  done
done
} > $O/c1.txt 2>&1
