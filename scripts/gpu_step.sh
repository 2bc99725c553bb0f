# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/g17; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > $O/pytest_wide.log 2>&1; echo "pytest exit $?" >> $O/pytest_wide.log
timeout 1800 python scripts/fig1_grid.py > $O/fig1_grid.jsonl 2>&1
timeout 500 python scripts/fuzz_gpu.py 420 140000 jit_mode=1,section_ops=150,group_tiles=3 > $O/fuzz_sections.json 2>&1
timeout 500 python scripts/fuzz_gpu.py 420 150000 jit_mode=2 > $O/fuzz_vm.json 2>&1
