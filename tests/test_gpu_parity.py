"""GPU parity: specialised sm_100a kernels (through the C ABI) vs the C oracle.

Bars (north star): int64 and interval bit-exact; fp64 strict mode bit-exact;
fp64 fused mode |gpu - ref| <= 1e-12 * sum_t |c_t| prod |x|^a (TOL below).
"""
import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W
import pyoracle

pytestmark = pytest.mark.gpu

TOL = 1e-12  # relative to the sum of absolute term magnitudes (north star)


def _dev(arrs, device):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(a)).to(device) for a in arrs]


def _f64_check(wl, n, device, strict_too=True):
    prog = pe.compile(wl.poly, wl.schemes)
    pts = wl.points(n)
    orc = pyoracle.Oracle(wl.poly, wl.schemes)
    ref = orc.eval_f64(pts)
    scale = pyoracle.abs_term_sum(wl.poly, pts)
    got = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(_dev(pts, device)).cpu().numpy()
    err = np.abs(got - ref)
    assert np.all(err <= TOL * scale), f"max rel err {np.max(err / scale):.3e}"
    if strict_too:
        gs = pe.Evaluator(pe.DoubleDomain(strict=True), prog).evaluate(_dev(pts, device)).cpu().numpy()
        assert np.array_equal(gs.view(np.int64), ref.view(np.int64)), "strict fp64 not bit-exact"
    return prog, pts, got


@pytest.mark.parametrize("degree,scheme", [(1000, "estrin"), (1000, "balanced"),
                                           (1023, "estrin"), (1023, "balanced")])
def test_c2_fp64(degree, scheme, cuda_device):
    _f64_check(W.c2(degree, scheme), 50_000, cuda_device)


def test_c1_horner_full_batch(cuda_device):
    wl = W.c1()
    _f64_check(wl, wl.n_points, cuda_device)  # the whole 1e5 batch


def test_c4_trivariate_sparse(cuda_device):
    _f64_check(W.c4(), 4_000, cuda_device)


def test_c3_int64_exact(cuda_device):
    wl = W.c3()
    prog = pe.compile(wl.poly, wl.schemes)
    pts = wl.points(200_000)
    ref = pyoracle.Oracle(wl.poly, wl.schemes).eval_i64(pts)
    got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate(_dev(pts, cuda_device)).cpu().numpy()
    assert np.array_equal(got, ref)


def test_c5_interval_bit_exact(cuda_device):
    wl = W.c5()
    prog = pe.compile(wl.poly, wl.schemes)
    lo, hi = wl.points(100_000)
    olo, ohi = pyoracle.Oracle(wl.poly, wl.schemes).eval_interval(lo, hi)
    glo, ghi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate(
        (_dev(lo, cuda_device), _dev(hi, cuda_device)))
    assert np.array_equal(glo.cpu().numpy(), olo)
    assert np.array_equal(ghi.cpu().numpy(), ohi)


def test_host_and_device_paths_identical(cuda_device):
    wl = W.c2(1000, "balanced")
    prog = pe.compile(wl.poly, wl.schemes)
    pts = wl.points(300_001)
    ev = pe.Evaluator(pe.DoubleDomain(), prog)
    host = ev.evaluate(pts)  # numpy -> staged H2D / walk / D2H pipeline
    dev = ev.evaluate(_dev(pts, cuda_device)).cpu().numpy()
    assert np.array_equal(host.view(np.int64), dev.view(np.int64))


EXAMPLE = ([8, 7, 6, 5, 4, 3, 2, 1, 0], [3, -1, 2, 1, -4, 9, -3, -2, 1])


@pytest.mark.parametrize("scheme", ["direct", "horner", "estrin", "balanced"])
def test_worked_example_all_domains(scheme, cuda_device):
    # reference eval_test.cpp:80-93: p(2)=793, p(0)=1, p(1)=6 for every scheme
    e, c = EXAMPLE
    pi = pe.Polynomial(np.array(e).reshape(-1, 1), np.array(c, dtype=np.int64))
    prog = pe.compile(pi, pe.builtin_scheme(scheme))
    got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate([np.array([2, 0, 1], dtype=np.int64)])
    assert list(got) == [793, 1, 6]
    gf = pe.Evaluator(pe.DoubleDomain(), prog).evaluate([np.array([2.0, 0.0, 1.0])])
    assert list(gf) == [793.0, 1.0, 6.0]
    lo, hi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate(
        ([np.array([2.0, 0.0, 1.0])], [np.array([2.0, 0.0, 1.0])]))
    assert np.all(lo <= np.array([793, 1, 6])) and np.all(hi >= np.array([793, 1, 6]))


def test_multivariate_example(cuda_device):
    # reference eval_test.cpp:95-107: x^2 y^2 + 2xy + 1 at (2,3) = 49
    p = pe.Polynomial(np.array([[2, 2], [1, 1], [0, 0]]), np.array([1, 2, 1], dtype=np.int64),
                      ("x", "y"))
    prog = pe.compile(p, [pe.builtin_scheme("horner")] * 2)
    got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate([np.array([2]), np.array([3])])
    assert list(got) == [49]


def test_float_point_cli_example(cuda_device):
    # reference cli_test.cpp:104-109: x^2+1 at 1.5 -> 3.25
    p = pe.Polynomial(np.array([[2], [0]]), np.array([1.0, 1.0]))
    prog = pe.compile(p, pe.builtin_scheme("balanced"))
    assert pe.Evaluator(pe.DoubleDomain(), prog).evaluate([np.array([1.5])])[0] == 3.25


def test_zero_polynomial(cuda_device):
    p = pe.Polynomial(np.zeros((0, 1), dtype=np.uint32), np.zeros(0, dtype=np.int64))
    prog = pe.compile(p, pe.builtin_scheme("estrin"))
    assert list(pe.Evaluator(pe.BigIntDomain(), prog).evaluate([np.array([17, -3])])) == [0, 0]


@pytest.mark.parametrize("n", [0, 1, 127, 128, 129, 4097])
def test_ragged_batch_sizes(n, cuda_device):
    wl = W.c2(1000, "estrin")
    prog = pe.compile(wl.poly, wl.schemes)
    pts = wl.points(n)
    ref = pyoracle.Oracle(wl.poly, wl.schemes).eval_f64(pts)
    got = pe.Evaluator(pe.DoubleDomain(strict=True), prog).evaluate(pts)
    assert got.shape == (n,)
    assert np.array_equal(got.view(np.int64), ref.view(np.int64))
