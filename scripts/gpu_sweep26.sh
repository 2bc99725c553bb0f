# C1 chain loop: rotating prefetch register sets (PE_LOOP_ROT=1) at depth 1..3
O=gpurun_out/sweep26; mkdir -p $O
for cfg in "0 1" "1 1" "1 2" "1 3"; do
  set -- $cfg
  export PE_LOOP_ROT=$1 PE_LOOP_DEPTH=$2
  timeout 600 python -m pytest tests/test_gpu_edges.py -x -q -k "chain" > $O/pytest_rot$1_d$2.log 2>&1; echo "exit $?" >> $O/pytest_rot$1_d$2.log
  r=$(timeout 600 python bench.py --config c1 --no-cpu --no-e2e --steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "c1 1e5 ROT=$1 DEPTH=$2 :: ms_per_step frac $r" >> $O/c1.txt
  r=$(timeout 600 python scripts/profile_one.py --config c1 --points 10000000 --reps 4 2>&1 | tail -1)
  echo "c1 1e7 ROT=$1 DEPTH=$2 :: $r" >> $O/c1.txt
done
