"""Runs the smoke pieces one at a time (argv[1] = piece) with progress prints,
so a hang is attributable; see scripts/gpu_step.sh."""
import faulthandler
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
faulthandler.dump_traceback_later(90, exit=True)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
from paper_1307_5655_b200 import workloads as W  # noqa: E402
import pyoracle  # noqa: E402


def say(*a):
    print(*a, flush=True)


piece = sys.argv[1]
dev = torch.device("cuda:0")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4099
wl = W.c2(1000, "estrin")
wl.poly = W.dense_univariate(200, W._rng(99))
pts = wl.points(n)
x = [torch.from_numpy(a).to(dev) for a in pts]
say("piece", piece, "n", n)
if piece == "f64vm":
    prog = pe.compile(wl.poly, wl.schemes)
    got = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(x).cpu().numpy()
    say("vm call done", got[:2])
    prog.compile_only(pe.DOMAIN_F64)
    say("compile_only done")
    got2 = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(x).cpu().numpy()
    say("kernel call done", np.array_equal(got.view(np.int64), got2.view(np.int64)))
elif piece.startswith("iv"):
    lo, hi = [pts[0]], [pts[0] + 1e-6]
    olo, ohi = pyoracle.Oracle(wl.poly, wl.schemes).eval_interval(lo, hi)
    prog = pe.compile(wl.poly, wl.schemes)
    tune = {"iv": dict(jit_mode=1), "ivsplit": dict(jit_mode=1, iv_partition_min=1, iv_partition=3),
            "ivclassify": dict(jit_mode=1, iv_partition_min=1),
            "ivnopart": dict(jit_mode=1, iv_partition=-1), "ivvm": dict(jit_mode=2)}[piece]
    prog.set_tuning(**tune)
    prog.compile_only(pe.DOMAIN_INTERVAL)
    say("compiled", "split" if "pe_walk_interval_split" in prog.ptx(pe.DOMAIN_INTERVAL) else "no split entry")
    glo, ghi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate(
        ([torch.from_numpy(lo[0]).to(dev)], [torch.from_numpy(hi[0]).to(dev)]))
    torch.cuda.synchronize()
    say("call done")
    glo, ghi = glo.cpu().numpy(), ghi.cpu().numpy()
    say("exact", np.array_equal(glo, olo), np.array_equal(ghi, ohi))
    bad = np.nonzero((glo.view(np.int64) != olo.view(np.int64)) | (ghi.view(np.int64) != ohi.view(np.int64)))[0]
    say("mismatches", len(bad), "first", bad[:16], "mod 512", bad[:16] % 512)
    for i in bad[:6]:
        say(i, "x", lo[0][i], "gpu", glo[i], ghi[i], "oracle", olo[i], ohi[i])
    if len(bad):
        say("bad x>0:", int(np.sum(lo[0][bad] > 0)), "bad x<0:", int(np.sum(hi[0][bad] < 0)),
            "blocks:", np.unique(bad // 512)[:20], "nblocks", len(np.unique(bad // 512)))
elif piece == "i64":
    w3 = W.c3()
    p3 = pe.compile(w3.poly, w3.schemes)
    p3.set_tuning(jit_mode=1)
    pts3 = w3.points(n)
    ref3 = pyoracle.Oracle(w3.poly, w3.schemes).eval_i64(pts3)
    got3 = pe.Evaluator(pe.BigIntDomain(), p3).evaluate([torch.from_numpy(a).to(dev) for a in pts3]).cpu().numpy()
    say("exact", np.array_equal(got3, ref3))
say("piece", piece, "ok")
