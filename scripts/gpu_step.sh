# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s26; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q --timeout 600 > $O/pytest_wide.log 2>&1; echo "pytest exit $?" >> $O/pytest_wide.log
for args in "64 1000 8192 balanced" "64 1000 8192 horner" "64 256 16384 balanced" "64 256 16384 horner" "64 64 65536 balanced" "2048 256 296 balanced" "2048 256 2048 balanced" "2048 256 2048 horner"; do
  timeout 300 python scripts/wide_profile.py $args >> $O/wide_kernel_only.jsonl 2>> $O/wide.err
done
