O=gpurun_out/verify
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c5 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --config c4 --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err
