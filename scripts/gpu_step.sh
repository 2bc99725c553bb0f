# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s34; mkdir -p $O
timeout 600 python scripts/fuzz_gpu.py 480 900000 jit_mode=1,lanes=2,block=128 > $O/fuzz_lanes2.json 2>&1
timeout 600 python scripts/fuzz_gpu.py 480 910000 jit_mode=1,chain_min=8,lanes=3 > $O/fuzz_chain8.json 2>&1
timeout 600 python scripts/fuzz_gpu.py 480 920000 jit_mode=1,sched_window=1,iv_mid=-1 > $O/fuzz_nosched.json 2>&1
timeout 600 python scripts/fuzz_gpu.py 480 930000 jit_mode=1,section_ops=64,group_tiles=1,iv_partition_min=1 > $O/fuzz_sections64.json 2>&1
