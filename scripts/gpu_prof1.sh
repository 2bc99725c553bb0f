set -x
python scripts/profile_one.py --config c2e1000 --reps 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pe_walk -s 1 -c 1 -o gpurun_out/prof_c2e python scripts/profile_one.py --config c2e1000 --reps 2 > gpurun_out/ncu_c2e.log 2>&1
echo "exit $?"
