O=gpurun_out/ncufinal; mkdir -p $O
python scripts/profile_one.py --config c4 --points 100000000 --reps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:pe_walk -s 4 -c 4 \
  -o $O/ncu_c4 python scripts/profile_one.py --config c4 --points 100000000 --reps 2 > $O/ncu_c4.log 2>&1
python scripts/profile_one.py --config c5 --points 100000000 --reps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"classify|pe_walk" -s 4 -c 4 \
  -o $O/ncu_c5 python scripts/profile_one.py --config c5 --points 100000000 --reps 2 > $O/ncu_c5.log 2>&1
