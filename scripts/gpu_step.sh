O=gpurun_out/g15; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for c in c4 c2 c3 c1 c5; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python bench.py --impl reference > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
timeout 2000 bash scripts/ncu_captures.sh c4 c5 c2e1000 c3
