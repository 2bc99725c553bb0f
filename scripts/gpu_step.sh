# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s5; mkdir -p $O
timeout 150 python scripts/debug_smoke.py ivsplit 200000 > $O/dbg_ivsplit_200k.log 2>&1; echo "exit $?" >> $O/dbg_ivsplit_200k.log
grep -q "exact True True" $O/dbg_ivsplit_200k.log || exit 1
timeout 500 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "interval or partition or 2_53" > $O/pytest_iv.log 2>&1; echo "pytest exit $?" >> $O/pytest_iv.log
timeout 600 python scripts/profile_one.py --config c5 --points 100000000 --reps 3 \
  --tune jit_mode=1 --tune jit_mode=1,iv_partition=2 > $O/c5_modes.jsonl 2> $O/c5_modes.err
scripts/probes/dfma_load_mix.bin > $O/dfma_load_mix.jsonl 2>&1
timeout 1500 python scripts/profile_one.py --config c4 --points 20000000 --reps 3 \
  --tune jit_mode=1 \
  --tune jit_mode=1,lanes=2,block=256 \
  --tune jit_mode=1,lanes=2,block=256,section_ops=1500 \
  --tune jit_mode=1,lanes=2,block=256,section_ops=2000 \
  --tune jit_mode=1,lanes=2,block=256,section_ops=4000 \
  --tune jit_mode=1,lanes=2,block=256,section_ops=6000 \
  --tune jit_mode=1,lanes=2,block=256,group_tiles=2 \
  --tune jit_mode=1,lanes=2,block=256,group_tiles=8 \
  --tune jit_mode=1,lanes=2,block=128 \
  --tune jit_mode=1,lanes=3,block=128 \
  --tune jit_mode=1,lanes=1,block=256 \
  --tune jit_mode=1,lanes=1,block=384 \
  > $O/c4_shapes.jsonl 2> $O/c4_shapes.err
for c in c2e1000 c2b1023; do
timeout 600 python scripts/profile_one.py --config $c --points 10000000 --reps 3 \
  --tune jit_mode=1 \
  --tune jit_mode=1,lanes=6 \
  --tune jit_mode=1,lanes=8 \
  --tune jit_mode=1,lanes=6,block=128 \
  --tune jit_mode=1,lanes=8,block=128,min_ctas=1 \
  --tune jit_mode=1,lanes=8,block=256,min_ctas=1 \
  --tune jit_mode=1,lanes=5 \
  >> $O/c2_shapes.jsonl 2>> $O/c2_shapes.err
done
timeout 600 python scripts/profile_one.py --config c1 --points 100000 --reps 20 \
  --tune jit_mode=1 --tune jit_mode=1,lanes=1,block=128 --tune jit_mode=1,lanes=2,block=128 \
  --tune jit_mode=1,lanes=1,block=256 --tune jit_mode=1,lanes=2,block=64 --tune jit_mode=1,lanes=1,block=64 \
  --tune jit_mode=1,lanes=2,block=256 \
  > $O/c1_shapes.jsonl 2> $O/c1_shapes.err
