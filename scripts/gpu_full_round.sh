#!/bin/bash
# Full measurement round on the GPU box (run through gpurun from the repo
# root after `python -c "import __graft_entry__ as g; g.build()"` here):
# smoke, GPU tests, bench per config + the reference arm, ncu launch lists
# and full captures, FP64 peaks, time to first result, the Figure-1 grid and
# a randomized parity sweep. Outputs under gpurun_out/round/ (copy the ones
# to keep into profiles/).
O=gpurun_out/round
mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for c in c4 c2 c3 c5 c1; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference > $O/bench_reference_c4.json 2> $O/bench_reference_c4.err
timeout 3000 bash scripts/ncu_captures.sh c4 c5 c5split c2e1000 c3
python scripts/fp64_peaks.py > $O/fp64_peaks.json 2>&1
[ -x scripts/probes/dfma_load_mix.bin ] || nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 \
  -o scripts/probes/dfma_load_mix.bin scripts/probes/dfma_load_mix.cu
scripts/probes/dfma_load_mix.bin > $O/probe_dfma_load_mix.jsonl 2>&1
for args in "64 1000 8192 balanced" "64 1000 8192 horner" "64 256 16384 balanced" "2048 256 2048 balanced"; do
  timeout 300 python scripts/wide_profile.py $args >> $O/wide_kernel_only.jsonl 2>> $O/wide.err
done
PE_CACHE_DIR=off timeout 900 python scripts/first_call.py > $O/first_call.jsonl 2>&1
timeout 700 python scripts/fuzz_gpu.py 600 600000 > $O/fuzz.json 2>&1
timeout 700 python scripts/fuzz_wide.py 600 700000 > $O/fuzz_wide.json 2>&1
timeout 2400 python scripts/fig1_grid.py > $O/fig1_grid.jsonl 2>&1
echo done > $O/DONE
