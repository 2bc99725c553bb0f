# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/g18; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "interval or c5 or vm or smoke or partition" > $O/pytest_iv.log 2>&1; echo "pytest exit $?" >> $O/pytest_iv.log
timeout 900 python bench.py --config c5 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err
timeout 1200 bash scripts/ncu_captures.sh c5
timeout 600 python scripts/fuzz_gpu.py 480 160000 > $O/fuzz.json 2>&1
