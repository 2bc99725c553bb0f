#!/bin/bash
# Final bench set on the final code (smoke + bench c1-c5 + reference arm).
O=gpurun_out/round8; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference > $O/bench_reference_c2.json 2> $O/bench_reference_c2.err
