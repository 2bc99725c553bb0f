# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s12; mkdir -p $O
timeout 1200 python scripts/profile_one.py --config c4 --points 20000000 --reps 3 \
  --tune jit_mode=1 \
  --tune jit_mode=1,lanes=2,block=384,section_ops=1500 \
  --tune jit_mode=1,lanes=2,block=384,section_ops=2500 \
  --tune jit_mode=1,lanes=2,block=512,section_ops=1600 \
  --tune jit_mode=1,lanes=2,block=320,section_ops=2000 \
  > $O/c4_shapes2.jsonl 2> $O/c4_shapes2.err
