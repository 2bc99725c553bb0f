"""GPU: programs imported from the reference's own compile() output
(pe_program_from_compiled) evaluate exactly like the ones built from terms,
and like the reference itself (int64 / interval / strict fp64 bit-exact)."""
import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W
import pyoracle

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not pyoracle.ref_available(), reason="oracle/_ref not built")]


def _t(a, device):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def _pair(wl):
    ref = pyoracle.Reference(wl.poly, wl.schemes)
    progs, sets = ref.export()
    return ref, pe.CompiledProgram.from_compiled(progs, sets, integer=wl.domain == "i64")


def test_f64_strict_and_fused(cuda_device):
    wl = W.c2(1000, "balanced")
    ref, prog = _pair(wl)
    pts = wl.points(50_003)
    want = ref.eval_f64(pts, 8)
    x = [_t(p, cuda_device) for p in pts]
    strict = pe.Evaluator(pe.DoubleDomain(strict=True), prog).evaluate(x).cpu().numpy()
    assert np.array_equal(strict.view(np.int64), want.view(np.int64))
    fused = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(x).cpu().numpy()
    assert np.all(np.abs(fused - want) <= 1e-12 * pyoracle.abs_term_sum(wl.poly, pts))


def test_int64_exact(cuda_device):
    wl = W.c3()
    ref, prog = _pair(wl)
    pts = wl.points(100_000)
    got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate([_t(p, cuda_device) for p in pts])
    assert np.array_equal(got.cpu().numpy(), ref.eval_i64(pts, 8))


def test_interval_bit_exact(cuda_device):
    wl = W.c5()
    ref, prog = _pair(wl)
    lo, hi = wl.points(100_000)
    glo, ghi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate(
        ([_t(a, cuda_device) for a in lo], [_t(a, cuda_device) for a in hi]))
    olo, ohi = ref.eval_interval(lo, hi, 8)
    assert np.array_equal(glo.cpu().numpy().view(np.int64), olo.view(np.int64))
    assert np.array_equal(ghi.cpu().numpy().view(np.int64), ohi.view(np.int64))


def test_trivariate_nested_unsliced(cuda_device):
    wl = W.c4()
    ref, prog = _pair(wl)
    pts = wl.points(20_000)
    got = pe.Evaluator(pe.DoubleDomain(), prog).evaluate([_t(p, cuda_device) for p in pts])
    want = ref.eval_f64(pts, 8)
    assert np.all(np.abs(got.cpu().numpy() - want) <= 1e-12 * pyoracle.abs_term_sum(wl.poly, pts))
