set -x
python scripts/profile_c2_all.py --reps 2 > gpurun_out/c2all_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pe_walk -s 4 -c 4 -o gpurun_out/prof_c2all python scripts/profile_c2_all.py --reps 2 > gpurun_out/ncu_c2all.log 2>&1
python scripts/profile_one.py --config c4 --reps 2 --points 4000000 > gpurun_out/c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pe_walk -s 6 -c 2 -o gpurun_out/prof_c4slices python scripts/profile_one.py --config c4 --reps 2 --points 4000000 > gpurun_out/ncu_c4.log 2>&1
echo done
