# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s32; mkdir -p $O
for c in c5 c3; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 700 python scripts/fuzz_gpu.py 600 500000 > $O/fuzz_a.json 2>&1
timeout 700 python scripts/fuzz_gpu.py 600 510000 jit_mode=1,iv_partition_min=1 > $O/fuzz_b.json 2>&1
timeout 700 python scripts/fuzz_gpu.py 600 520000 jit_mode=1,iv_partition=3,iv_partition_min=1 > $O/fuzz_c.json 2>&1
timeout 700 python scripts/fuzz_gpu.py 600 530000 jit_mode=1,section_ops=200,group_tiles=3 > $O/fuzz_d.json 2>&1
