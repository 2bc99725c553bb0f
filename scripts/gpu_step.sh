O=gpurun_out/g10; mkdir -p $O
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --impl reference > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
timeout 1500 bash scripts/ncu_captures.sh c4
