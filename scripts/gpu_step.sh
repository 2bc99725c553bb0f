O=gpurun_out/g16; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_wide.py tests/test_gpu_edges.py -x -q -k "wide or sliced or section" > $O/pytest_wide.log 2>&1; echo "pytest exit $?" >> $O/pytest_wide.log
timeout 1500 python scripts/fig1_grid.py --quick > $O/fig1_quick.jsonl 2>&1
timeout 2000 bash scripts/ncu_captures.sh c4 c2e1000 c3
