O=gpurun_out/sweep14; mkdir -p $O
python scripts/fuzz_repro.py 40191 40238 > $O/repro.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -k "partition or interval" > $O/pytest_part.log 2>&1; echo "exit $?" >> $O/pytest_part.log
{
for m in 0 1; do
  r=$(PE_IV_PART=$m timeout 600 python scripts/profile_one.py --config c5 --points 10000000 --reps 4 2>&1 | tail -1)
  echo "c5 1e7 PE_IV_PART=$m :: $r"
  r=$(PE_IV_PART=$m timeout 600 python scripts/profile_one.py --config c5 --points 100000000 --reps 3 2>&1 | tail -1)
  echo "c5 1e8 PE_IV_PART=$m :: $r"
done
} > $O/c5.txt 2>&1
timeout 900 python bench.py --config c5 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err
