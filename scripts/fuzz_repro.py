"""Replays one fuzz_gpu.py seed and, for the interval domain, compares every
kernel mode with the oracle: python scripts/fuzz_repro.py <seed> [tuning]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "scripts")]
import numpy as np  # noqa: E402

import fuzz_gpu as F  # noqa: E402
import paper_1307_5655_b200 as pe  # noqa: E402
import pyoracle  # noqa: E402

seed = int(sys.argv[1])
base = {"jit_mode": 1}
if len(sys.argv) > 2:
    base = {k: int(v) for k, v in (kv.split("=") for kv in sys.argv[2].split(",") if kv)}
rng = np.random.default_rng(seed)
integer = bool(rng.random() < 0.35)
p = F.poly(rng, integer)
sch = [F.scheme(rng) for _ in range(p.nvars)]
n = int(rng.choice([1, 33, 1000, 4099]))
print("seed", seed, "integer", integer, "nvars", p.nvars, "terms", len(p.coefficients), "n", n,
      "schemes", [(int(s.upper), int(s.lower), int(s.cutoff)) for s in sch],
      "max exp", p.exponents.max(axis=0).tolist(), flush=True)
if integer:
    span = int(rng.choice([2, 3, 10, 200]))
    xi = [rng.integers(-span, span + 1, n).astype(np.int64) for _ in range(p.nvars)]
x = [F.points(rng, n) for _ in range(p.nvars)]
w = [np.abs(a) * 10.0 ** rng.uniform(-17, 0, n) * (rng.random(n) < 0.7) for a in x]
lo = [a.copy() for a in x]
hi = [a + b for a, b in zip(x, w)]
for v in range(p.nvars):
    m = rng.random(n) < 0.05
    lo[v][m] = -np.abs(hi[v][m])
    bad = ~(lo[v] <= hi[v])
    lo[v][bad], hi[v][bad] = 0.0, 0.0
orc = pyoracle.Oracle(p, sch)
with np.errstate(all="ignore"):
    olo, ohi = orc.eval_interval(lo, hi)
modes = {"given": base, "default": {"jit_mode": 1}, "no partition": {"jit_mode": 1, "iv_partition": -1},
         "strict replay": {"jit_mode": 1, "iv_fast": -1}, "no mid": {"jit_mode": 1, "iv_mid": -1},
         "vm": {"jit_mode": 2}, "split": {"jit_mode": 1, "iv_partition": 3, "iv_partition_min": 1},
         "partmin1": {"jit_mode": 1, "iv_partition_min": 1}}
for name, tune in modes.items():
    prog = pe.compile(p, sch)
    prog.set_tuning(**tune)
    with np.errstate(all="ignore"):
        glo, ghi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate((lo, hi))
    badi = np.nonzero((glo.view(np.int64) != olo.view(np.int64)) | (ghi.view(np.int64) != ohi.view(np.int64)))[0]
    print(f"{name:14s} mismatches {len(badi)}", badi[:8].tolist(), flush=True)
    for i in badi[:4]:
        print("   i", i, "in", [(float(l[i]).hex(), float(h[i]).hex()) for l, h in zip(lo, hi)],
              "gpu", float(glo[i]).hex(), float(ghi[i]).hex(), "oracle", float(olo[i]).hex(), float(ohi[i]).hex())
if pyoracle.ref_available():
    rlo, rhi = pyoracle.Reference(p, sch).eval_interval(lo, hi)
    print("oracle == reference:", bool(np.array_equal(rlo.view(np.int64), olo.view(np.int64))
                                        and np.array_equal(rhi.view(np.int64), ohi.view(np.int64))))
