"""Per-call cost of a small batch (C1: Hörner d1000, 1e5 points, device
buffers): kernel time (CUDA events around 200 back-to-back launches), host
time per Evaluator.evaluate call, host time of the bare C-ABI call with
pre-built arguments, and one isolated call timed like bench.py."""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
from paper_1307_5655_b200 import _lib as L  # noqa: E402
from paper_1307_5655_b200 import workloads as W  # noqa: E402

n = int(os.environ.get("N", "100000"))
wl = W.c1()
prog = pe.compile(wl.poly, wl.schemes)
ev = pe.Evaluator(pe.DoubleDomain(), prog, device=0)
x = torch.from_numpy(wl.points(n)[0]).cuda()
out = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream() if os.environ.get("SIDE_STREAM") else torch.cuda.current_stream()
ev.evaluate([x], out=out, stream=s.cuda_stream)
torch.cuda.synchronize()

R = 200
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(R):
    ev.evaluate([x], out=out, stream=s.cuda_stream)
b.record(s)
torch.cuda.synchronize()
gpu_us = a.elapsed_time(b) * 1e3 / R

t = time.perf_counter()
for _ in range(R):
    ev.evaluate([x], out=out, stream=s.cuda_stream)
host_us = (time.perf_counter() - t) * 1e6 / R
torch.cuda.synchronize()

lib = L.lib()
ptrs = (C.c_void_p * 1)(x.data_ptr())
ex = ev._exec(s.cuda_stream)
optr = C.c_void_p(out.data_ptr())
t = time.perf_counter()
for _ in range(R):
    lib.pe_eval_f64(prog.handle, ptrs, n, optr, C.byref(ex))
capi_us = (time.perf_counter() - t) * 1e6 / R
torch.cuda.synchronize()

iso = []
for _ in range(20):
    torch.cuda.synchronize()
    a.record(s)
    ev.evaluate([x], out=out, stream=s.cuda_stream)
    b.record(s)
    torch.cuda.synchronize()
    iso.append(a.elapsed_time(b) * 1e3)
iso.sort()
print(json.dumps({"n": n, 
                  "stream": "side" if os.environ.get("SIDE_STREAM") else "current(default)",
                  "gpu_us_per_call_back_to_back": round(gpu_us, 2),
                  "host_us_per_evaluate": round(host_us, 2),
                  "host_us_per_capi_call": round(capi_us, 2),
                  "isolated_call_us_median": round(iso[len(iso) // 2], 2),
                  "kernel_stats": prog.kernel_stats(pe.DOMAIN_F64)}))
