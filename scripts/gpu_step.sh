# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s28; mkdir -p $O
for c in c2e1000 c2b1000 c2e1023 c2b1023 c3; do
timeout 600 python scripts/profile_one.py --config $c --points 10000000 --reps 5 \
  --tune jit_mode=1 --tune jit_mode=1,regbound_smem=1 >> $O/regbound.jsonl 2>> $O/regbound.err
done
timeout 300 python scripts/profile_one.py --config c2e1000 --strict --points 10000000 --reps 5 \
  --tune jit_mode=1 --tune jit_mode=1,regbound_smem=1 >> $O/regbound.jsonl 2>> $O/regbound.err
