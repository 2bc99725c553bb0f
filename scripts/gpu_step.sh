O=gpurun_out/g8; mkdir -p $O
T="--tune section_ops=4294967295"
for s in 1000 2000 3000; do for g in 4 16; do T="$T --tune section_ops=$s,group_tiles=$g"; done; done
T="$T --tune section_ops=1000,group_tiles=16,sched_window=1 --tune section_ops=1500,group_tiles=16 --tune section_ops=700,group_tiles=16"
timeout 900 python scripts/profile_one.py --config c4 --points 100000000 --reps 2 $T > $O/c4_sweep.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q -k "section" > $O/pytest_sec.log 2>&1; echo "pytest exit $?" >> $O/pytest_sec.log
