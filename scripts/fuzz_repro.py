"""Re-runs fuzz_gpu.check(seed) for given seeds under several kernel modes
(subprocess per mode, so codegen env vars apply) and, for the default mode,
prints the first mismatching intervals.

  python scripts/fuzz_repro.py SEED [SEED ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "scripts")]

MODES = {"default": {}, "mid0": {"PE_IV_MID": "0"}, "fast0": {"PE_IV_FAST": "0"},
         "part_min1": {"PE_IV_PART_MIN": "1"}, "part0": {"PE_IV_PART": "0"},
         "signs0": {"PE_IV_SIGNS": "0"}, "imm2": {"PE_IMM": "2"}}

if len(sys.argv) > 2 and sys.argv[1] == "--one":
    import numpy as np
    import fuzz_gpu as F
    seed = int(sys.argv[2])
    import paper_1307_5655_b200 as pe
    orig = pe.Evaluator.evaluate

    def spy(self, x, *a, **k):
        out = orig(self, x, *a, **k)
        if isinstance(x, tuple):
            spy.last = (x, out)
        return out
    pe.Evaluator.evaluate = spy
    try:
        F.check(seed)
        print("PASS")
    except AssertionError as e:
        print("FAIL", e)
        if os.environ.get("DIAG") and hasattr(spy, "last"):
            (lo, hi), (glo, ghi) = spy.last
            rng_prog = np.random.default_rng(seed)
            import pyoracle
            # recompute the oracle on the same inputs
            p_sch = F.poly(np.random.default_rng(seed), False)  # not used: print inputs only
            olo_ohi = None
            glo, ghi = np.asarray(glo), np.asarray(ghi)
            print("nvars", len(lo), "n", len(lo[0]))
            print("first points lo/hi:", [(float(lo[v][0]), float(hi[v][0])) for v in range(len(lo))])
            np.savez(f"gpurun_out/repro_{seed}.npz", *(list(lo) + list(hi)), glo=glo, ghi=ghi)
    sys.exit(0)

for seed in sys.argv[1:]:
    for name, env in MODES.items():
        e = dict(os.environ, **env)
        if name == "default":
            e["DIAG"] = "1"
        r = subprocess.run([sys.executable, __file__, "--one", seed], env=e, capture_output=True,
                           text=True, timeout=900)
        print(f"seed {seed} {name}: {(r.stdout.strip() or r.stderr.strip()[-300:])}")
