# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s14; mkdir -p $O
timeout 150 python scripts/debug_smoke.py ivsplit 4099 > $O/dbg_ivsplit_4k.log 2>&1; echo "exit $?" >> $O/dbg_ivsplit_4k.log
timeout 150 python scripts/debug_smoke.py ivsplit 1000003 > $O/dbg_ivsplit_1m.log 2>&1; echo "exit $?" >> $O/dbg_ivsplit_1m.log
grep -q "exact True True" $O/dbg_ivsplit_1m.log || exit 1
timeout 600 python scripts/profile_one.py --config c5 --points 100000000 --reps 3 \
  --tune jit_mode=1 --tune jit_mode=1,iv_partition=3 --tune jit_mode=1,iv_partition=3,block=256 \
  --tune jit_mode=1,iv_partition=3,sync_every=64 --tune jit_mode=1,iv_partition=3,sync_every=16 \
  --tune jit_mode=1,iv_partition=3,sync_every=128 > $O/c5_modes.jsonl 2> $O/c5_modes.err
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "partition" > $O/pytest_part.log 2>&1; echo "pytest exit $?" >> $O/pytest_part.log
