set -x
PE_LANES=6 python scripts/profile_one.py --config c2e1000 --reps 3 > gpurun_out/prof_plain.log 2>&1 && \
PE_LANES=3 python scripts/profile_one.py --config c4 --points 4000000 --reps 3 >> gpurun_out/prof_plain.log 2>&1 && \
python -c "
import ctypes as C, sys; sys.path.insert(0,'.')
from paper_1307_5655_b200 import _lib as L
for k in (0,1):
    v=C.c_double(); s=C.c_int32(); L.check(L.lib().pe_measure_peak(0,k,C.byref(v),C.byref(s))); print('peak kind',k, v.value/1e12, 'T ops/s', s.value)
" >> gpurun_out/prof_plain.log 2>&1 && \
PE_LANES=6 ncu --set full --clock-control none --import-source on -k regex:pe_walk -s 1 -c 1 -o gpurun_out/prof_c2e_L6 python scripts/profile_one.py --config c2e1000 --reps 2 > gpurun_out/ncu1.log 2>&1
PE_LANES=3 ncu --set full --clock-control none --import-source on -k regex:pe_walk -s 1 -c 1 -o gpurun_out/prof_c4_L3 python scripts/profile_one.py --config c4 --points 4000000 --reps 2 > gpurun_out/ncu2.log 2>&1
echo "exit $?"
