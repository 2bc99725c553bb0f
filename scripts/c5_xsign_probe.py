"""Bounds the gain of a sign-partitioned interval fast path: C5 program on
1e7 intervals with x > 0 only, evaluated by the default kernel and by the
probe kernel that assumes positive coordinates (PE_IV_XSIGN=1, exact for
these inputs only). Prints both times and whether the results agree."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1:
    import numpy as np
    import torch
    import paper_1307_5655_b200 as pe
    from paper_1307_5655_b200 import workloads as W
    wl = W.c5()
    lo, hi = wl.points(10_000_000)
    lo = [np.abs(lo[0]) + 1e-3]
    hi = [lo[0] + 1e-6]
    x = ([torch.from_numpy(lo[0]).cuda()], [torch.from_numpy(hi[0]).cuda()])
    ev = pe.Evaluator(pe.IntervalDomain(), pe.compile(wl.poly, wl.schemes), deferred_checks=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(4):
        a.record()
        out = ev.evaluate(x)
        b.record()
        torch.cuda.synchronize()
        ev.synchronize()
    np.save(sys.argv[1], torch.stack(out).cpu().numpy())
    print(f"{a.elapsed_time(b):.3f}")
    sys.exit(0)
import numpy as np  # noqa: E402
ts = {}
for xs in ("0", "1"):
    env = dict(os.environ, PE_IV_XSIGN=xs)
    ts[xs] = subprocess.run([sys.executable, __file__, f"/tmp/xs{xs}.npy"], env=env,
                            capture_output=True, text=True).stdout.strip()
same = np.array_equal(np.load("/tmp/xs0.npy").view(np.int64), np.load("/tmp/xs1.npy").view(np.int64))
print(f"default {ts['0']} ms, positive-x probe {ts['1']} ms, identical={same}")
