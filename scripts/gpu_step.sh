O=gpurun_out/g12; mkdir -p $O
python scripts/fp64_peaks.py > $O/peaks.json 2>&1
nvidia-smi -q -d CLOCK > $O/clocks.txt 2>&1
T=""
for s in 500 1000 2000; do T="$T --tune lanes=2,block=256,section_ops=$s --tune lanes=2,block=384,section_ops=$s"; done
T="$T --tune section_ops=3000,group_tiles=2 --tune section_ops=3000,group_tiles=3 --tune section_ops=2500 --tune section_ops=3500"
timeout 1500 python scripts/profile_one.py --config c4 --points 100000000 --reps 2 $T > $O/c4_sweep.jsonl 2>&1
