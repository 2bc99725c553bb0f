O=gpurun_out/g14; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -k "interval or c5 or vm or smoke" > $O/pytest_iv.log 2>&1; echo "pytest exit $?" >> $O/pytest_iv.log
timeout 700 python scripts/fuzz_gpu.py 480 130000 > $O/fuzz.json 2>&1
timeout 900 python bench.py --config c5 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err
PE_CACHE_DIR=off timeout 900 python scripts/first_call.py > $O/first_call.jsonl 2>&1
