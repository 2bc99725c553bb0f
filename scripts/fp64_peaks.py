"""FP64 pipe vs FP64 tensor cores on this GPU:
DFMA/s (FMA pipe), DMMA FMA/s (mma.sync m8n8k4 f64), int64 MAD/s and the
dependent-DFMA latency, through pe_measure_peak. One JSON line."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1307_5655_b200 import _lib as L  # noqa: E402

out = {}
for kind, name in ((0, "dfma_fma_per_s"), (3, "dmma_fma_per_s"), (1, "imad64_per_s"),
                   (2, "dfma_latency_cycles")):
    v, sms = C.c_double(), C.c_int32()
    L.check(L.lib().pe_measure_peak(0, kind, C.byref(v), C.byref(sms)))
    out[name] = v.value
out["sms"] = sms.value
out["dmma_over_dfma"] = out["dmma_fma_per_s"] / out["dfma_fma_per_s"]
print(json.dumps(out))
