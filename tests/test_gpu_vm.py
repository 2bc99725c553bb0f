"""Walk VM (runtime/vm_kernels.cu): the ahead-of-time interpreter that answers
a new program's first calls while its specialised kernel compiles.

Bars: the VM runs the specialised kernel's op sequence, so its results equal
the specialised kernel bit for bit in every domain (and therefore meet the
oracle bars: int64 / interval / strict fp64 bit-exact, fused fp64 within
1e-12 * sum|terms|). jit_mode 0 (the library default) answers the first call
with the VM and switches to the compiled kernel once the background compile
finishes; the first call of a fresh d1000 program needs no ptxas run.
"""
import time

import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W
import pyoracle

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _dev(arrs, device):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(a)).to(device) for a in arrs]


def _pair(wl, **tune):
    vm = pe.compile(wl.poly, wl.schemes)
    vm.set_tuning(jit_mode=2, **tune)
    jit = pe.compile(wl.poly, wl.schemes)
    jit.set_tuning(jit_mode=1, **tune)
    return vm, jit


def _bits(a):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    return a.view(np.int64)


@pytest.mark.parametrize("make", [W.c1, lambda: W.c2(1000, "estrin"), lambda: W.c2(1023, "balanced"),
                                  W.c4])
@pytest.mark.parametrize("strict", [False, True])
def test_vm_fp64_equals_kernel_and_oracle(make, strict, cuda_device):
    wl = make()
    n = 20_011 if wl.name.startswith("C4") else 100_003
    pts = wl.points(n)
    vm, jit = _pair(wl)
    x = _dev(pts, cuda_device)
    a = pe.Evaluator(pe.DoubleDomain(strict=strict), vm).evaluate(x)
    b = pe.Evaluator(pe.DoubleDomain(strict=strict), jit).evaluate(x)
    assert np.array_equal(_bits(a), _bits(b))
    ref = pyoracle.Oracle(wl.poly, wl.schemes).eval_f64(pts)
    if strict:
        assert np.array_equal(_bits(a), ref.view(np.int64))
    else:
        scale = pyoracle.abs_term_sum(wl.poly, pts)
        assert np.all(np.abs(a.cpu().numpy() - ref) <= TOL * scale)


@pytest.mark.parametrize("int_pipe", [False, True])
def test_vm_int64_exact(int_pipe, cuda_device):
    wl = W.c3()
    pts = wl.points(50_021)
    vm, jit = _pair(wl)
    x = _dev(pts, cuda_device)
    dom = pe.BigIntDomain(int_pipe=int_pipe)
    a = pe.Evaluator(dom, vm).evaluate(x).cpu().numpy()
    b = pe.Evaluator(dom, jit).evaluate(x).cpu().numpy()
    ref = pyoracle.Oracle(wl.poly, wl.schemes).eval_i64(pts)
    assert np.array_equal(a, ref) and np.array_equal(b, ref)
    # the range check still flags coordinates beyond the proven bound
    big = [p.copy() for p in pts]
    big[0][17] = 2**40
    with pytest.raises(OverflowError):
        pe.Evaluator(pe.BigIntDomain(int_pipe=int_pipe), vm).evaluate(big, bounds=[2, 2])


def test_vm_interval_bit_exact_on_edge_cases(cuda_device):
    rng = np.random.default_rng(77)
    n = 30_000
    for scheme, deg in (("estrin", 200), ("horner", 31), ("balanced", 64)):
        p = pe.Polynomial(np.arange(deg, -1, -1).reshape(-1, 1), rng.uniform(-1, 1, deg + 1))
        x = rng.uniform(-1, 1, n)
        lo, hi = x.copy(), x + 1e-6
        lo[:40], hi[:40] = -1e-3, 1e-3            # straddles zero
        lo[40:60], hi[40:60] = 0.0, 0.5           # touches zero
        lo[60:80], hi[60:80] = 1e-310, 2e-310     # subnormal
        lo[80:100], hi[80:100] = 1e200, 1e201     # overflow to inf
        lo[100:110], hi[100:110] = -np.inf, 1.0   # infinite endpoint
        wl = W.Workload("iv", p, [pe.builtin_scheme(scheme)], "interval", n, 0)
        vm, jit = _pair(wl)
        args = ([_dev([lo], cuda_device)[0]], [_dev([hi], cuda_device)[0]])
        a = pe.Evaluator(pe.IntervalDomain(), vm).evaluate(args)
        b = pe.Evaluator(pe.IntervalDomain(), jit).evaluate(args)
        o = pyoracle.Oracle(p, [pe.builtin_scheme(scheme)]).eval_interval([lo], [hi])
        for g, k, r in zip(a, b, o):
            assert np.array_equal(_bits(g), r.view(np.int64)), scheme
            assert np.array_equal(_bits(k), r.view(np.int64)), scheme


def test_vm_host_buffers_and_invalid_intervals(cuda_device):
    wl = W.c5()
    vm, _ = _pair(wl)
    lo, hi = wl.points(70_001)
    got = pe.Evaluator(pe.IntervalDomain(), vm).evaluate((lo, hi))
    o = pyoracle.Oracle(wl.poly, wl.schemes).eval_interval([lo[0][:3000]], [hi[0][:3000]])
    for g, r in zip(got, o):
        assert np.array_equal(np.asarray(g)[:3000].view(np.int64), r.view(np.int64))
    bad = lo[0].copy()
    bad[5] = hi[0][5] + 1.0
    with pytest.raises(ValueError):
        pe.Evaluator(pe.IntervalDomain(), vm).evaluate(([bad], hi))


def test_first_call_runs_vm_then_switches_to_kernel(cuda_device, monkeypatch):
    # jit_mode 0 (library default): a fresh program's first call is answered
    # by the VM without waiting for ptxas; the specialised kernel compiles in
    # the background and later calls use it — same bits either way
    import torch
    monkeypatch.setenv("PE_CACHE_DIR", "off")  # no cubin from an earlier run
    wl = W.c2(1000, "balanced")
    pts = wl.points(100_000)
    x = _dev(pts, cuda_device)
    # warm the CUDA context and the VM module on another program
    warm = pe.compile(pe.Polynomial(np.array([[2], [0]]), np.array([1.0, 1.0])),
                      pe.builtin_scheme("horner"))
    warm.set_tuning(jit_mode=2)
    pe.Evaluator(pe.DoubleDomain(), warm).evaluate(x[:1])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prog = pe.compile(wl.poly, wl.schemes)
    prog.set_tuning(jit_mode=0)
    first = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(x)
    torch.cuda.synchronize()
    first_s = time.perf_counter() - t0
    assert first_s < 0.25, f"first call took {first_s:.3f} s"
    prog.compile_only(pe.DOMAIN_F64)  # waits for the background compile
    assert prog.kernel_ready(pe.DOMAIN_F64)
    later = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(x)
    assert np.array_equal(_bits(first), _bits(later))
    ref = pyoracle.Oracle(wl.poly, wl.schemes).eval_f64(pts)
    assert np.all(np.abs(later.cpu().numpy() - ref) <= TOL * pyoracle.abs_term_sum(wl.poly, pts))
