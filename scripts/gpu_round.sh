python -c "
import ctypes as C, sys; sys.path.insert(0,'.')
from paper_1307_5655_b200 import _lib as L
v=C.c_double(); s=C.c_int32()
L.check(L.lib().pe_measure_peak(0,2,C.byref(v),C.byref(s))); print('dfma latency cycles', v.value)
L.check(L.lib().pe_measure_peak(0,0,C.byref(v),C.byref(s))); print('dfma peak', v.value/1e12)
" > gpurun_out/lat.log 2>&1
timeout 600 python scripts/e2e_chunks.py > gpurun_out/e2e_chunks.log 2>&1
