"""BASELINE.json sizes on the GPU, checked through size-independent
properties: a deterministic subsample against the C oracle (every k-th point
plus both ends and the shard boundaries of an 8-way split), shard invariance
(the 8-GPU split evaluated slice by slice gives identical bits), and
determinism across calls."""
import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W
from paper_1307_5655_b200.shard import shard_bounds
import pyoracle

pytestmark = pytest.mark.gpu


def _sample_idx(n, count=2000, world=8):
    idx = set(np.linspace(0, n - 1, count).astype(np.int64).tolist())
    for r in range(world):
        s, e = shard_bounds(n, world, r)
        idx.update([s, max(s, e - 1)])
    idx.update([0, 1, n - 2, n - 1])
    return np.array(sorted(i for i in idx if 0 <= i < n))


def _shards_equal(evaluate, cols, n, full):
    import torch
    parts = []
    for r in range(8):
        s, e = shard_bounds(n, 8, r)
        parts.append(evaluate([c[s:e] for c in cols]))
    return torch.equal(torch.cat(parts), full)


@pytest.mark.parametrize("degree,scheme", [(1000, "estrin"), (1023, "balanced")])
def test_c2_full_batch(degree, scheme, cuda_device):
    import torch
    wl = W.c2(degree, scheme)
    prog = pe.compile(wl.poly, wl.schemes)
    pts = wl.points()
    n = wl.n_points
    cols = [torch.from_numpy(a).to(cuda_device) for a in pts]
    ev = pe.Evaluator(pe.DoubleDomain(), prog)
    out = ev.evaluate(cols)
    idx = _sample_idx(n)
    sub = [a[idx] for a in pts]
    ref = pyoracle.Oracle(wl.poly, wl.schemes).eval_f64(sub)
    scale = pyoracle.abs_term_sum(wl.poly, sub)
    got = out.cpu().numpy()[idx]
    assert np.all(np.abs(got - ref) <= 1e-12 * scale)
    assert _shards_equal(ev.evaluate, cols, n, out)
    assert torch.equal(ev.evaluate(cols), out)


def test_c3_full_batch(cuda_device):
    import torch
    wl = W.c3()
    prog = pe.compile(wl.poly, wl.schemes)
    pts = wl.points()
    n = wl.n_points
    cols = [torch.from_numpy(a).to(cuda_device) for a in pts]
    ev = pe.Evaluator(pe.BigIntDomain(), prog)
    out = ev.evaluate(cols)
    idx = _sample_idx(n, 20_000)
    ref = pyoracle.Oracle(wl.poly, wl.schemes).eval_i64([a[idx] for a in pts])
    assert np.array_equal(out.cpu().numpy()[idx], ref)
    assert _shards_equal(ev.evaluate, cols, n, out)


def test_c4_full_batch(cuda_device):
    import torch
    wl = W.c4()
    prog = pe.compile(wl.poly, wl.schemes)
    n = wl.n_points  # 1e8 points, 2.4 GB of coordinates
    pts = wl.points()
    cols = [torch.from_numpy(a).to(cuda_device) for a in pts]
    ev = pe.Evaluator(pe.DoubleDomain(), prog)
    out = ev.evaluate(cols)
    idx = _sample_idx(n, 600)
    sub = [a[idx] for a in pts]
    ref = pyoracle.Oracle(wl.poly, wl.schemes).eval_f64(sub)
    scale = pyoracle.abs_term_sum(wl.poly, sub)
    assert np.all(np.abs(out.cpu().numpy()[idx] - ref) <= 1e-12 * scale)
    assert _shards_equal(ev.evaluate, cols, n, out)


def test_c5_full_batch(cuda_device):
    import torch
    wl = W.c5()
    prog = pe.compile(wl.poly, wl.schemes)
    n = wl.n_points
    lo, hi = wl.points()
    dlo = [torch.from_numpy(lo[0]).to(cuda_device)]
    dhi = [torch.from_numpy(hi[0]).to(cuda_device)]
    ev = pe.Evaluator(pe.IntervalDomain(), prog)
    olo, ohi = ev.evaluate((dlo, dhi))
    idx = _sample_idx(n, 20_000)
    # include the points the fast path hands to the fixup kernel (|x| tiny)
    tiny = np.nonzero(np.abs(lo[0][:2_000_000]) < 4e-3)[0][:2000]
    idx = np.unique(np.concatenate([idx, tiny]))
    rlo, rhi = pyoracle.Oracle(wl.poly, wl.schemes).eval_interval([lo[0][idx]], [hi[0][idx]])
    assert np.array_equal(olo.cpu().numpy()[idx], rlo)
    assert np.array_equal(ohi.cpu().numpy()[idx], rhi)
    parts_lo, parts_hi = [], []
    for r in range(8):
        s, e = shard_bounds(n, 8, r)
        a, b = ev.evaluate(([dlo[0][s:e]], [dhi[0][s:e]]))
        parts_lo.append(a)
        parts_hi.append(b)
    assert torch.equal(torch.cat(parts_lo), olo) and torch.equal(torch.cat(parts_hi), ohi)
