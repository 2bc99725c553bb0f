#!/bin/bash
# ncu --set full captures of every config's dominant kernel(s) at the bench's
# own launch sizes (one GPU, after the same commands ran clean without ncu).
O=gpurun_out/ncu
mkdir -p $O
python scripts/profile_one.py --config c1 --points 100000 --reps 2 > /dev/null && \
ncu --set full --import-source on --clock-control none -k regex:pe_walk -s 1 -c 1 \
  -o $O/ncu_c1 python scripts/profile_one.py --config c1 --points 100000 --reps 2 > $O/c1.log 2>&1
python scripts/profile_one.py --config c4 --points 100000000 --reps 1 > /dev/null && \
ncu --set full --import-source on --clock-control none -k regex:pe_walk -s 6 -c 6 \
  -o $O/ncu_c4 python scripts/profile_one.py --config c4 --points 100000000 --reps 2 > $O/c4.log 2>&1
python scripts/profile_one.py --config c5 --points 100000000 --reps 1 > /dev/null && \
ncu --set full --import-source on --clock-control none -k regex:pe_walk_interval$ -s 1 -c 1 \
  -o $O/ncu_c5 python scripts/profile_one.py --config c5 --points 100000000 --reps 2 > $O/c5.log 2>&1
echo done > $O/DONE
