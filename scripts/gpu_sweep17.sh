# C1: bench with steps enqueued back to back; chain-loop prefetch depth.
O=gpurun_out/sweep17; mkdir -p $O
{
for d in 1 2 3; do
  r=$(PE_LOOP_DEPTH=$d timeout 600 python bench.py --config c1 --no-cpu --no-e2e --steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "c1 1e5 LOOP_DEPTH=$d :: ms_per_step frac $r"
  r=$(PE_LOOP_DEPTH=$d timeout 600 python scripts/profile_one.py --config c1 --points 10000000 --reps 4 2>&1 | tail -1)
  echo "c1 1e7 LOOP_DEPTH=$d :: $r"
done
} > $O/c1.txt 2>&1
timeout 900 python bench.py --config c2 --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
