"""e2e (pinned host buffers) of the four C2 programs via pe_eval_f64_multi for
several staging chunk sizes (PE_STAGE_CHUNK is read per call)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W
wls = W.c2_all()
progs = [pe.compile(w.poly, w.schemes) for w in wls]
x = [torch.from_numpy(a).pin_memory() for a in wls[0].points()]
outs = [torch.empty(x[0].shape[0], dtype=torch.float64).pin_memory() for _ in wls]
xs = [a.numpy() for a in x]
os_ = [o.numpy() for o in outs]
chunks = [int(c) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else \
    [0, 1 << 18, 1 << 19, 625000, 1 << 21, 1250000]
for chunk in chunks:
    if chunk:
        os.environ["PE_STAGE_CHUNK"] = str(chunk)
    else:
        os.environ.pop("PE_STAGE_CHUNK", None)
    pe.evaluate_many(progs, xs, outs=os_)
    t = time.perf_counter()
    for _ in range(5):
        pe.evaluate_many(progs, xs, outs=os_)
    el = (time.perf_counter() - t) / 5
    print(f"slots={os.environ.get('PE_STAGE_SLOTS', 3)} chunk={chunk or 'default'}: "
          f"{el * 1e3:.2f} ms/step -> {4e7 / el:.3e} points/s", flush=True)
