# Scratch: the command of the most recent gpurun call (see gpu_full_round.sh for a full round).
O=gpurun_out/s29; mkdir -p $O
for sch in balanced horner; do
ncu --set full --import-source on --clock-control none -k regex:wide_walk -s 1 -c 1 \
  -o $O/ncu_wide_$sch python scripts/wide_profile.py 64 1000 8192 $sch > $O/ncu_$sch.log 2>&1
ncu -i $O/ncu_wide_$sch.ncu-rep --page raw --csv > $O/r2_ncu_wide_${sch}_raw.csv 2>/dev/null
ncu -i $O/ncu_wide_$sch.ncu-rep --page details --csv > $O/r2_ncu_wide_${sch}_details.csv 2>/dev/null
rm -f $O/ncu_wide_$sch.ncu-rep
done
timeout 700 python scripts/fuzz_gpu.py 600 400000 > $O/fuzz_default.json 2>&1
timeout 700 python scripts/fuzz_gpu.py 600 410000 jit_mode=1,section_ops=200,group_tiles=3 > $O/fuzz_sections.json 2>&1
timeout 700 python scripts/fuzz_gpu.py 600 420000 jit_mode=2 > $O/fuzz_vm.json 2>&1
