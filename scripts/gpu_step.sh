# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s13; mkdir -p $O
timeout 900 python -m pytest tests/test_bench_ranks.py -m gpu -q --timeout 600 > $O/pytest_ranks.log 2>&1; echo "pytest exit $?" >> $O/pytest_ranks.log
for c in c4 c2 c3 c5 c1; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --config c5 --tune iv_partition=3 > $O/bench_c5_split.json 2> $O/bench_c5_split.err
timeout 500 python scripts/fuzz_gpu.py 420 300000 jit_mode=1,iv_partition=3,iv_partition_min=1 > $O/fuzz_split.json 2>&1
timeout 500 python scripts/fuzz_gpu.py 420 310000 jit_mode=1,iv_partition_min=1 > $O/fuzz_partmin1.json 2>&1
