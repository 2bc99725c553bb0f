# C1 (1e5 points, L2 flushed per step): constant-cache warm-up of the
# chain-loop arrays (PE_WARM 0 none / 1 prefetchu / 2 per-thread ld.const).
O=gpurun_out/sweep12; mkdir -p $O
{
for w in 0 1 2; do
  for L in 4 2 1; do
    r=$(PE_WARM=$w PE_LANES=$L timeout 600 python bench.py --config c1 --no-cpu --no-e2e --steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")
    echo "c1 1e5 PE_WARM=$w LANES=$L :: ms_per_step frac $r"
  done
  r=$(PE_WARM=$w timeout 600 python scripts/profile_one.py --config c1 --points 10000000 --reps 4 2>&1 | tail -1)
  echo "c1 1e7 PE_WARM=$w :: $r"
done
} > $O/c1.txt 2>&1
