O=gpurun_out/g5; mkdir -p $O
T=""
for s in 1000 2000 3000; do for g in 2 8 32; do T="$T --tune section_ops=$s,group_tiles=$g,sched_window=1 --tune section_ops=$s,group_tiles=$g"; done; done
timeout 900 python scripts/profile_one.py --config c4 --points 4000000 --reps 3 $T > $O/c4_sweep.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -k "section" > $O/pytest_sec.log 2>&1; echo "pytest exit $?" >> $O/pytest_sec.log
