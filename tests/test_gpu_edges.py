"""GPU edge cases: exact-integer tiers and overflow refusal, invalid intervals,
special values, host/device pointer handling, determinism."""
import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W
import pyoracle

pytestmark = pytest.mark.gpu


def _t(a, device):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def test_i64_fp64_tier_equals_int_pipe(cuda_device):
    wl = W.c3()
    prog = pe.compile(wl.poly, wl.schemes)
    pts = wl.points(100_003)
    a = pe.Evaluator(pe.BigIntDomain(), prog).evaluate([_t(p, cuda_device) for p in pts])
    b = pe.Evaluator(pe.BigIntDomain(int_pipe=True), prog).evaluate([_t(p, cuda_device) for p in pts])
    ref = pyoracle.Oracle(wl.poly, wl.schemes).eval_i64(pts)
    assert np.array_equal(a.cpu().numpy(), ref) and np.array_equal(b.cpu().numpy(), ref)


def test_i64_large_values_use_int_pipe_exactly(cuda_device):
    # values far above 2^53 but below 2^63: only the int64 kernel is exact
    p = pe.Polynomial(np.array([[3], [1], [0]]), np.array([7, -3, 2**40], dtype=np.int64))
    prog = pe.compile(p, pe.builtin_scheme("horner"))
    x = np.array([2**17 + 5, -(2**17) - 11, 3, 0, 123456], dtype=np.int64)
    got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate([x])
    ref = [7 * int(v) ** 3 - 3 * int(v) + 2**40 for v in x]
    assert [int(g) for g in got] == ref


def test_i64_retry_with_actual_maxima(cuda_device):
    # uniform bound is limited by y^30; x far above it still provably fits
    p = pe.Polynomial(np.array([[1, 0], [0, 30]]), np.array([1, 1], dtype=np.int64), ("x", "y"))
    prog = pe.compile(p, [pe.builtin_scheme("balanced")] * 2)
    x = np.array([2**40, -(2**40), 5], dtype=np.int64)
    y = np.array([2, -2, 1], dtype=np.int64)
    got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate([_t(x, cuda_device), _t(y, cuda_device)])
    assert [int(v) for v in got.cpu().numpy()] == [int(a) + int(b) ** 30 for a, b in zip(x, y)]


def test_i64_overflow_is_refused(cuda_device):
    p = pe.Polynomial(np.array([[40]]), np.array([3], dtype=np.int64))
    prog = pe.compile(p, pe.builtin_scheme("estrin"))
    with pytest.raises(OverflowError):
        pe.Evaluator(pe.BigIntDomain(), prog).evaluate([np.array([1, 2, 4], dtype=np.int64)])
    # INT64_MIN coordinate can never satisfy a bound
    with pytest.raises(OverflowError):
        pe.Evaluator(pe.BigIntDomain(), prog).evaluate([np.array([np.iinfo(np.int64).min])])


def test_i64_caller_bounds(cuda_device):
    wl = W.c3()
    prog = pe.compile(wl.poly, wl.schemes)
    ev = pe.Evaluator(pe.BigIntDomain(), prog)
    pts = wl.points(1000)
    ref = pyoracle.Oracle(wl.poly, wl.schemes).eval_i64(pts)
    assert np.array_equal(ev.evaluate(pts, bounds=[2, 2]), ref)
    with pytest.raises(OverflowError):  # asserted bound violated by the data
        ev.evaluate(pts, bounds=[1, 1])
    with pytest.raises(OverflowError):  # proof impossible for the asserted range
        ev.evaluate(pts, bounds=[1 << 40, 1 << 40])


def test_interval_rejects_invalid_endpoints(cuda_device):
    wl = W.c5()
    prog = pe.compile(wl.poly, wl.schemes)
    ev = pe.Evaluator(pe.IntervalDomain(), prog)
    with pytest.raises(ValueError):
        ev.evaluate(([np.array([0.5, 2.0])], [np.array([0.6, 1.0])]))  # lo > hi
    with pytest.raises(ValueError):
        ev.evaluate(([np.array([np.nan])], [np.array([1.0])]))


def test_interval_special_values_bit_exact(cuda_device):
    specials = np.array([0.0, -0.0, 5e-324, -5e-324, 2.2250738585072014e-308, 1e-300, -1e-300, 1.0,
                         -1.0, 1e154, -1e154, 1e300, -1e300, 1.7976931348623157e308,
                         -1.7976931348623157e308, np.inf, -np.inf])
    lo = np.minimum.outer(specials, specials).ravel()
    hi = np.maximum.outer(specials, specials).ravel()
    rng = np.random.default_rng(9)
    for scheme in ("horner", "estrin", "balanced", "direct"):
        c = rng.uniform(-1, 1, 13)
        p = pe.Polynomial(np.arange(12, -1, -1).reshape(-1, 1), c)
        prog = pe.compile(p, pe.builtin_scheme(scheme))
        glo, ghi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate(([lo], [hi]))
        olo, ohi = pyoracle.Oracle(p, [pe.builtin_scheme(scheme)]).eval_interval([lo], [hi])
        assert np.array_equal(glo.view(np.int64), olo.view(np.int64))
        assert np.array_equal(ghi.view(np.int64), ohi.view(np.int64))


def test_f64_special_values_strict_bit_exact(cuda_device):
    x = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1e308, -1e308, 1e-200])
    p = pe.Polynomial(np.arange(7, -1, -1).reshape(-1, 1), np.linspace(-1, 1, 8))
    for scheme in ("horner", "estrin", "balanced"):
        prog = pe.compile(p, pe.builtin_scheme(scheme))
        got = pe.Evaluator(pe.DoubleDomain(strict=True), prog).evaluate([x])
        ref = pyoracle.Oracle(p, [pe.builtin_scheme(scheme)]).eval_f64([x])
        same = (got.view(np.int64) == ref.view(np.int64)) | (np.isnan(got) & np.isnan(ref))
        assert same.all()


def test_arity_mismatch(cuda_device):
    prog = pe.compile(W.c3().poly, W.c3().schemes)
    with pytest.raises(ValueError):
        pe.Evaluator(pe.BigIntDomain(), prog).evaluate([np.array([1], dtype=np.int64)])


def test_repeatable_and_shard_invariant(cuda_device):
    # the walk is per point: evaluating halves separately gives identical bits
    import torch
    wl = W.c4()
    prog = pe.compile(wl.poly, wl.schemes)
    pts = [_t(a, cuda_device) for a in wl.points(20_001)]
    ev = pe.Evaluator(pe.DoubleDomain(), prog)
    full = ev.evaluate(pts)
    again = ev.evaluate(pts)
    halves = torch.cat([ev.evaluate([a[:7777] for a in pts]), ev.evaluate([a[7777:] for a in pts])])
    assert torch.equal(full, again) and torch.equal(full, halves)


@pytest.mark.parametrize("mid", [0, -1])
def test_interval_fast_path_equals_strict_replay(cuda_device, mid):
    # The fast interval path (sign-case products, FP64-pipe nextafter with
    # "did not move" checks, static signs) and the fixup replay (with and
    # without its finite-case stage) must equal the strict replay and the
    # oracle on intervals that straddle zero, touch zero, underflow and
    # overflow.
    rng = np.random.default_rng(21)
    n = 50_000
    x = rng.uniform(-1, 1, n)
    w = np.where(rng.uniform(size=n) < 0.1, rng.uniform(0, 0.5, n), 1e-6)
    lo, hi = x.copy(), x + w
    lo[:50] = 0.0                      # touches zero from above
    hi[:50] = np.abs(hi[:50])
    hi[50:100] = 0.0                   # touches zero from below
    lo[50:100] = -np.abs(lo[50:100])
    lo[100:150] = -np.abs(hi[100:150])  # straddles zero
    hi[100:150] = np.abs(hi[100:150])
    big = rng.uniform(1e150, 1e160, 200)
    lo[200:400], hi[200:400] = big, big * 2
    tiny = rng.uniform(1e-200, 1e-190, 200)
    lo[400:600], hi[400:600] = tiny, tiny * 2
    for scheme, deg in (("estrin", 200), ("horner", 30), ("balanced", 64)):
        wl = W.c5()
        p = pe.Polynomial(np.arange(deg, -1, -1).reshape(-1, 1), rng.uniform(-1, 1, deg + 1))
        slow = pe.compile(p, pe.builtin_scheme(scheme))
        slow.set_tuning(iv_fast=-1)
        s = pe.Evaluator(pe.IntervalDomain(), slow).evaluate(([lo], [hi]))
        fast = pe.compile(p, pe.builtin_scheme(scheme))
        fast.set_tuning(iv_mid=mid)
        f = pe.Evaluator(pe.IntervalDomain(), fast).evaluate(([lo], [hi]))
        assert "%facc" not in slow.ptx(pe.DOMAIN_INTERVAL)
        assert "%facc" in fast.ptx(pe.DOMAIN_INTERVAL)
        o = pyoracle.Oracle(p, [pe.builtin_scheme(scheme)]).eval_interval([lo], [hi])
        for a, b, c in zip(f, s, o):
            assert np.array_equal(a.view(np.int64), c.view(np.int64))
            assert np.array_equal(b.view(np.int64), c.view(np.int64))


def test_deferred_checks_same_results_and_late_errors(cuda_device):
    import torch
    w3, w5 = W.c3(), W.c5()
    p3, p5 = pe.compile(w3.poly, w3.schemes), pe.compile(w5.poly, w5.schemes)
    x3 = [_t(a, cuda_device) for a in w3.points(70_001)]
    lo, hi = w5.points(70_001)
    x5 = ([_t(lo[0], cuda_device)], [_t(hi[0], cuda_device)])
    e3 = pe.Evaluator(pe.BigIntDomain(), p3, deferred_checks=True)
    e5 = pe.Evaluator(pe.IntervalDomain(), p5, deferred_checks=True)
    a3, (a5l, a5h) = e3.evaluate(x3), e5.evaluate(x5)
    e3.synchronize()
    b3 = pe.Evaluator(pe.BigIntDomain(), p3).evaluate(x3)
    b5l, b5h = pe.Evaluator(pe.IntervalDomain(), p5).evaluate(x5)
    assert torch.equal(a3, b3) and torch.equal(a5l, b5l) and torch.equal(a5h, b5h)
    # a bound violation surfaces at synchronize(), not at the call
    bad = [x3[0].clone(), x3[1].clone()]
    bad[0][5] = 1 << 40
    e3.evaluate(bad)
    with pytest.raises(OverflowError):
        e3.synchronize()
    e3.synchronize()  # status was reset
    badlo = x5[0][0].clone()
    badlo[3] = 5.0  # lo > hi
    e5.evaluate(([badlo], x5[1]))
    with pytest.raises(ValueError):
        e5.synchronize()


def test_evaluate_many_matches_single_calls(cuda_device):
    progs = [pe.compile(w.poly, w.schemes) for w in W.c2_all()]
    pts = W.c2(1000, "estrin").points(250_001)
    many_host = pe.evaluate_many(progs, pts)
    many_dev = pe.evaluate_many(progs, [_t(a, cuda_device) for a in pts])
    for p, h, d in zip(progs, many_host, many_dev):
        single = pe.Evaluator(pe.DoubleDomain(), p).evaluate(pts)
        assert np.array_equal(h.view(np.int64), single.view(np.int64))
        assert np.array_equal(d.cpu().numpy().view(np.int64), single.view(np.int64))


@pytest.mark.parametrize("section_ops", [2**32 - 1, 1000, 400])
@pytest.mark.parametrize("tiles", [1, 3, 8])
def test_sectioned_wide_program_bit_identical(cuda_device, section_ops, tiles):
    # long walks run as a persistent sectioned kernel (groups of tiles per
    # section pass, live values through scratch, coordinates reloaded, powers
    # rebuilt); the op sequence is unchanged, so every section count and
    # group size gives the unsectioned kernel's bits — within the fused
    # tolerance of the oracle, host or device buffers, ragged batch
    rng = np.random.default_rng(4)
    ex = np.unique(rng.integers(0, 20, size=(3000, 3)), axis=0).astype(np.uint32)
    p = pe.Polynomial(ex, rng.normal(size=len(ex)), ("x", "y", "z"))
    sch = [pe.builtin_scheme("balanced")] * 3
    pts = [rng.uniform(-1, 1, 10_007) for _ in range(3)]
    one = pe.compile(p, sch)
    one.set_tuning(section_ops=2**32 - 1)
    base = pe.Evaluator(pe.DoubleDomain(), one).evaluate([_t(a, cuda_device) for a in pts]).cpu().numpy()
    prog = pe.compile(p, sch)
    prog.set_tuning(section_ops=section_ops, group_tiles=tiles)
    if section_ops < 2**32 - 1:
        assert prog.f64_slices() > 1
    ref = pyoracle.Oracle(p, sch).eval_f64(pts)
    scale = pyoracle.abs_term_sum(p, pts)
    ev = pe.Evaluator(pe.DoubleDomain(), prog)
    dev = ev.evaluate([_t(a, cuda_device) for a in pts]).cpu().numpy()
    host = ev.evaluate(pts)
    assert np.all(np.abs(dev - ref) <= 1e-12 * scale)
    assert np.array_equal(dev.view(np.int64), host.view(np.int64))
    assert np.array_equal(dev.view(np.int64), base.view(np.int64))


@pytest.mark.parametrize("domain", ["f64strict", "i64"])
def test_sectioned_exact_domains(cuda_device, domain):
    # sections in the bit-exact domains: strict fp64 equals the oracle's
    # reference op order bit for bit, int64 is exact
    rng = np.random.default_rng(8)
    ex = np.unique(rng.integers(0, 12, size=(1500, 3)), axis=0).astype(np.uint32)
    sch = [pe.builtin_scheme("balanced")] * 3
    if domain == "i64":
        p = pe.Polynomial(ex, rng.integers(-8, 9, size=len(ex)).astype(np.int64), ("x", "y", "z"))
        pts = [rng.integers(-2, 3, 5003).astype(np.int64) for _ in range(3)]
        prog = pe.compile(p, sch)
        prog.set_tuning(section_ops=300)
        got = pe.Evaluator(pe.BigIntDomain(int_pipe=True), prog).evaluate(pts)
        assert np.array_equal(got, pyoracle.Oracle(p, sch).eval_i64(pts))
    else:
        p = pe.Polynomial(ex, rng.normal(size=len(ex)), ("x", "y", "z"))
        pts = [rng.uniform(-1, 1, 5003) for _ in range(3)]
        prog = pe.compile(p, sch)
        prog.set_tuning(section_ops=300)
        got = pe.Evaluator(pe.DoubleDomain(strict=True), prog).evaluate(pts)
        ref = pyoracle.Oracle(p, sch).eval_f64(pts)
        assert np.array_equal(got.view(np.int64), ref.view(np.int64))


@pytest.mark.parametrize("domain", ["f64", "i64", "interval"])
def test_no_out_of_bounds_writes(cuda_device, domain):
    # compute-sanitizer is closed on this pool: check the tail handling
    # directly — results for n points land in [0, n) and the canary words
    # after them (and before them) stay untouched, for ragged n and every
    # kernel shape (lanes x block) the runtime may pick
    import torch
    rng = np.random.default_rng(3)
    if domain == "i64":
        p = W.c3().poly
        sch = W.c3().schemes
    else:
        p = pe.Polynomial(np.arange(300, -1, -1).reshape(-1, 1), rng.uniform(-1, 1, 301))
        sch = [pe.builtin_scheme("estrin")]
    prog = pe.compile(p, sch)
    for n in (1, 31, 33, 127, 1025, 4097, 70_001):
        pad = 64
        dt = torch.int64 if domain == "i64" else torch.float64
        canary = 1 << 62 if domain == "i64" else 1e300  # no result can equal it
        outs = [torch.full((n + 2 * pad,), canary, dtype=dt, device=cuda_device)
                for _ in range(2 if domain == "interval" else 1)]
        if domain == "i64":
            cols = [torch.from_numpy(rng.integers(-2, 3, n)).to(cuda_device) for _ in range(p.nvars)]
            pe.Evaluator(pe.BigIntDomain(), prog).evaluate(cols, out=outs[0][pad:pad + n])
        elif domain == "f64":
            cols = [torch.from_numpy(rng.uniform(-1, 1, n)).to(cuda_device)]
            pe.Evaluator(pe.DoubleDomain(), prog).evaluate(cols, out=outs[0][pad:pad + n])
        else:
            lo = torch.from_numpy(rng.uniform(-1, 1, n)).to(cuda_device)
            pe.Evaluator(pe.IntervalDomain(), prog).evaluate(
                ([lo], [lo + 1e-6]), out=(outs[0][pad:pad + n], outs[1][pad:pad + n]))
        for o in outs:
            o = o.cpu()
            assert bool((o[:pad] == canary).all()) and bool((o[pad + n:] == canary).all()), n
            assert not bool((o[pad:pad + n] == canary).any()), n


def test_wide_univariate_program_is_sliced(cuda_device):
    # dense degree 20000: sliced into ~2k-record kernels (slice k holds the
    # terms of one exponent range; its tree has a large root partial degree)
    rng = np.random.default_rng(12)
    d = 20_000
    p = pe.Polynomial(np.arange(d, -1, -1).reshape(-1, 1), rng.uniform(-1, 1, d + 1))
    sch = [pe.builtin_scheme("estrin")]
    prog = pe.compile(p, sch)
    assert prog.f64_slices() > 1
    x = [rng.uniform(-1, 1, 3001)]
    got = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(x)
    ref = pyoracle.Oracle(p, sch).eval_f64(x)
    scale = pyoracle.abs_term_sum(p, x)
    assert np.all(np.abs(got - ref) <= 1e-12 * scale)


def test_program_shared_across_host_threads(cuda_device):
    # reference contract (eval.hpp:59-68): a compiled program is immutable and
    # shareable; sessions may run concurrently. Here 6 host threads share one
    # program (kernels JIT-compiled once), each on its own stream or host path.
    import threading
    import torch
    wl = W.c2(1000, "balanced")
    prog = pe.compile(wl.poly, wl.schemes)
    pts = wl.points(200_003)
    want = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(pts)
    results, errors = {}, []

    def work(i):
        try:
            if i % 2:
                results[i] = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(pts)
            else:
                s = torch.cuda.Stream(device=cuda_device)
                with torch.cuda.stream(s):
                    cols = [torch.from_numpy(a).to(cuda_device) for a in pts]
                    out = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(cols, stream=s.cuda_stream)
                    s.synchronize()
                results[i] = out.cpu().numpy()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for r in results.values():
        assert np.array_equal(r.view(np.int64), want.view(np.int64))


@pytest.mark.parametrize("n", [1, 31, 100_000, 100_003])
def test_chain_loop_bit_identical_to_straight_line(n, cuda_device):
    # the looped Hörner chain issues the same FMA sequence as the straight-line
    # kernel: results must agree bit for bit (and stay within TOL of the oracle)
    wl = W.c1()
    pts = wl.points(n)
    looped = pe.compile(wl.poly, wl.schemes)
    assert "$Lrun0" in looped.ptx(pe.DOMAIN_F64)
    a = pe.Evaluator(pe.DoubleDomain(), looped).evaluate([_t(pts[0], cuda_device)]).cpu().numpy()
    flat = pe.compile(wl.poly, wl.schemes)
    flat.set_tuning(chain_min=2**32 - 1)
    assert "$Lrun0" not in flat.ptx(pe.DOMAIN_F64)
    b = pe.Evaluator(pe.DoubleDomain(), flat).evaluate([_t(pts[0], cuda_device)]).cpu().numpy()
    assert np.array_equal(a.view(np.int64), b.view(np.int64))
    ref = pyoracle.Oracle(wl.poly, wl.schemes).eval_f64(pts)
    assert np.all(np.abs(a - ref) <= 1e-12 * pyoracle.abs_term_sum(wl.poly, pts))


def test_chain_loop_int64_exact(cuda_device):
    rng = np.random.default_rng(5)
    d = 150
    p = pe.Polynomial(np.arange(d, -1, -1).reshape(-1, 1),
                      rng.choice([-8, -3, -1, 1, 2, 7], d + 1).astype(np.int64))
    schemes = [pe.builtin_scheme("horner")]
    prog = pe.compile(p, schemes)
    assert "$Lrun0" in prog.ptx(pe.DOMAIN_I64)
    x = rng.integers(-1, 2, 20_011).astype(np.int64)
    ref = pyoracle.Oracle(p, schemes).eval_i64([x])
    for int_pipe in (False, True):  # exact-on-FP64 tier and int64 IMAD kernel
        got = pe.Evaluator(pe.BigIntDomain(int_pipe=int_pipe), prog).evaluate(
            [_t(x, cuda_device)]).cpu().numpy()
        assert np.array_equal(got, ref)


def test_sparse_horner_with_loop_tail(cuda_device):
    e = np.array([300, 299, 298] + list(range(200, -1, -1))).reshape(-1, 1)
    rng = np.random.default_rng(9)
    c = rng.uniform(-1, 1, len(e))
    schemes = [pe.builtin_scheme("horner")]
    poly = pe.Polynomial(e, c)
    prog = pe.compile(poly, schemes)
    x = [rng.uniform(-1.1, 1.1, 5000)]
    got = pe.Evaluator(pe.DoubleDomain(), prog).evaluate([_t(x[0], cuda_device)]).cpu().numpy()
    ref = pyoracle.Oracle(poly, schemes).eval_f64(x)
    assert np.all(np.abs(got - ref) <= 1e-12 * pyoracle.abs_term_sum(poly, x))


@pytest.mark.parametrize("scheme", ["horner", "estrin", "balanced", "direct"])
def test_interval_fast_path_extreme_magnitudes(scheme, cuda_device):
    # The fast interval path tracks operand signs statically (coefficients,
    # even powers, same-sign sums) and steps known-sign endpoints on the
    # integer pipe; coefficients from 1e-300 to 1e300 and points from
    # subnormal to 1e150 drive products through underflow to 0 / subnormals
    # and overflow to inf, where those shortcuts must hand over to the strict
    # replay. Bit-exact against the oracle.
    rng = np.random.default_rng(21)
    exps = np.array([[a, b] for a in range(0, 9) for b in range(0, 9 - a)
                     if rng.random() < 0.7], dtype=np.uint32)
    mags = 10.0 ** rng.uniform(-300, 300, len(exps))
    coefs = mags * rng.choice([-1.0, 1.0], len(exps))
    poly = pe.Polynomial(exps, coefs, ("x", "y"))
    schemes = [pe.builtin_scheme(scheme)] * 2
    prog = pe.compile(poly, schemes)
    n = 20_000
    cols_lo, cols_hi = [], []
    for _ in range(2):
        centre = rng.choice([-1.0, 1.0], n) * 10.0 ** rng.uniform(-320, 150, n)
        width = np.abs(centre) * 10.0 ** rng.uniform(-17, 0, n)
        lo, hi = centre, centre + width
        straddle = rng.random(n) < 0.05
        lo = np.where(straddle, -np.abs(hi), lo)
        cols_lo.append(np.minimum(lo, hi))
        cols_hi.append(np.maximum(lo, hi))
    glo, ghi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate(
        ([_t(c, cuda_device) for c in cols_lo], [_t(c, cuda_device) for c in cols_hi]))
    olo, ohi = pyoracle.Oracle(poly, schemes).eval_interval(cols_lo, cols_hi)
    glo, ghi = glo.cpu().numpy(), ghi.cpu().numpy()
    assert np.array_equal(glo.view(np.int64), olo.view(np.int64))
    assert np.array_equal(ghi.view(np.int64), ohi.view(np.int64))


def test_multi_device_host_batches_shard_and_gather(cuda_device):
    # pe_exec.devices: contiguous slices per listed device, results gathered
    # into the host output. One GPU on the box: the list repeats device 0
    # (each slice still runs its own pipeline); results must equal the
    # single-device call bit for bit.
    import torch
    ndev = torch.cuda.device_count()
    devs = list(range(ndev)) if ndev > 1 else [0, 0, 0]
    wl = W.c2(1000, "balanced")
    prog = pe.compile(wl.poly, wl.schemes)
    pts = wl.points(1_000_003)
    one = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(pts)
    many = pe.Evaluator(pe.DoubleDomain(), prog, devices=devs).evaluate(pts)
    assert np.array_equal(one.view(np.int64), many.view(np.int64))
    outs = pe.evaluate_many([prog, prog], pts, devices=devs)
    assert np.array_equal(outs[1].view(np.int64), one.view(np.int64))

    w3 = W.c3()
    p3 = pe.compile(w3.poly, w3.schemes)
    x3 = w3.points(300_001)
    assert np.array_equal(pe.Evaluator(pe.BigIntDomain(), p3, devices=devs).evaluate(x3),
                          pe.Evaluator(pe.BigIntDomain(), p3).evaluate(x3))

    w5 = W.c5()
    p5 = pe.compile(w5.poly, w5.schemes)
    lo, hi = w5.points(300_007)
    a = pe.Evaluator(pe.IntervalDomain(), p5, devices=devs).evaluate((lo, hi))
    b = pe.Evaluator(pe.IntervalDomain(), p5).evaluate((lo, hi))
    assert np.array_equal(a[0].view(np.int64), b[0].view(np.int64))
    assert np.array_equal(a[1].view(np.int64), b[1].view(np.int64))

    with pytest.raises(ValueError):  # device buffers live on one device
        pe.Evaluator(pe.DoubleDomain(), prog, devices=devs).evaluate(
            [_t(pts[0][:1000], cuda_device)])


def test_evaluate_parallel_and_register_check(cuda_device):
    # reference evaluate_parallel is bit-identical to evaluate for any worker
    # count (eval.hpp:91-96); the register check passes on compiled programs
    wl = W.c2(1000, "balanced")
    prog = pe.compile(wl.poly, wl.schemes)
    pts = wl.points(10_007)
    ev = pe.Evaluator(pe.DoubleDomain(strict=True), prog)
    ev.enable_register_check(True)
    a = ev.evaluate(pts)
    for w in (1, 3, 64):
        b = ev.evaluate_parallel(pts, w)
        assert np.array_equal(a.view(np.int64), b.view(np.int64))
    c = pe.evaluate_parallel(prog, pts, pe.DoubleDomain(strict=True), 4)
    assert np.array_equal(a.view(np.int64), c.view(np.int64))


def test_chain_loops_inside_nested_programs(cuda_device):
    # bivariate Hörner: each y-program is a 150-step chain (a loop), nested
    # inside the x-chain; f64 fused within tolerance, strict bit-exact, and
    # the int64 domain exact
    rng = np.random.default_rng(77)
    ex = np.array([(i, j) for i in range(4) for j in range(151)], dtype=np.uint32)
    schemes = [pe.builtin_scheme("horner")] * 2
    pf = pe.Polynomial(ex, rng.uniform(-1, 1, len(ex)), ("x", "y"))
    prog = pe.compile(pf, schemes)
    assert prog.ptx(pe.DOMAIN_F64).count("bra.uni $Lrun") == 4
    x = [rng.uniform(-1, 1, 5003), rng.uniform(-1, 1, 5003)]
    orc = pyoracle.Oracle(pf, schemes)
    ref = orc.eval_f64(x)
    got = pe.Evaluator(pe.DoubleDomain(), prog).evaluate([_t(a, cuda_device) for a in x]).cpu().numpy()
    assert np.all(np.abs(got - ref) <= 1e-12 * pyoracle.abs_term_sum(pf, x))
    pi = pe.Polynomial(ex, rng.choice([-3, -1, 1, 2, 5], len(ex)).astype(np.int64), ("x", "y"))
    prog_i = pe.compile(pi, schemes)
    assert "$Lrun" in prog_i.ptx(pe.DOMAIN_I64)
    xi = [rng.integers(-1, 2, 5003).astype(np.int64) for _ in range(2)]
    want = pyoracle.Oracle(pi, schemes).eval_i64(xi)
    for int_pipe in (False, True):
        got = pe.Evaluator(pe.BigIntDomain(int_pipe=int_pipe), prog_i).evaluate(
            [_t(a, cuda_device) for a in xi]).cpu().numpy()
        assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [1, 5, 33, 4097, 150_001])
@pytest.mark.parametrize("scheme", ["estrin", "horner", "balanced"])
@pytest.mark.parametrize("mode", ["split", "classify"])
def test_interval_sign_partition_bit_exact(n, scheme, mode, cuda_device):
    # Sign-partitioned fast path: x > 0 intervals run the program, x < 0
    # intervals the mirrored program q(y) = p(-y) at -x, the rest (touching /
    # straddling zero, invalid) the fixup replay — either in one kernel that
    # packs each CTA's intervals by sign in shared memory ("split",
    # iv_partition=3) or through the classifier kernel and two gathered
    # entries (the default).
    # Results must equal the unpartitioned kernel and the oracle bit for
    # bit, for every list length (empty lists, partial CTAs, ragged tails).
    rng = np.random.default_rng(1000 + n)
    deg = {"estrin": 200, "horner": 37, "balanced": 64}[scheme]
    p = pe.Polynomial(np.arange(deg, -1, -1).reshape(-1, 1), rng.uniform(-1, 1, deg + 1))
    x = rng.uniform(-1, 1, n)
    w = np.where(rng.uniform(size=n) < 0.05, rng.uniform(0, 0.3, n), 1e-6)
    lo, hi = x.copy(), x + w
    k = min(n, 40)
    lo[: k // 4] = 0.0                         # touches zero
    hi[: k // 4] = np.abs(hi[: k // 4]) + 1e-9
    lo[k // 4: k // 2] = -np.abs(lo[k // 4: k // 2])
    hi[k // 4: k // 2] = -0.0                  # negative side touching -0
    if n > 100:
        lo[50:60], hi[50:60] = 1e-200, 2e-200  # tiny positive: underflow -> fixup
        lo[60:70], hi[60:70] = -2e-200, -1e-200
        lo[70:80], hi[70:80] = 1e150, 2e150    # overflow
        lo[80:90], hi[80:90] = -2e150, -1e150
    part = pe.compile(p, pe.builtin_scheme(scheme))
    part.set_tuning(iv_partition_min=1, iv_partition=3 if mode == "split" else 0)
    f = pe.Evaluator(pe.IntervalDomain(), part).evaluate(([_t(lo, cuda_device)], [_t(hi, cuda_device)]))
    entry = "pe_walk_interval_pos" if mode == "classify" else "pe_walk_interval_split"
    assert entry in part.ptx(pe.DOMAIN_INTERVAL)
    plain = pe.compile(p, pe.builtin_scheme(scheme))
    plain.set_tuning(iv_partition=-1)
    g = pe.Evaluator(pe.IntervalDomain(), plain).evaluate(([_t(lo, cuda_device)], [_t(hi, cuda_device)]))
    assert "pe_walk_interval_pos" not in plain.ptx(pe.DOMAIN_INTERVAL)
    assert "pe_walk_interval_split" not in plain.ptx(pe.DOMAIN_INTERVAL)
    o = pyoracle.Oracle(p, [pe.builtin_scheme(scheme)]).eval_interval([lo], [hi])
    for a, b, c in zip(f, g, o):
        a, b = a.cpu().numpy(), b.cpu().numpy()
        assert np.array_equal(a.view(np.int64), c.view(np.int64))
        assert np.array_equal(b.view(np.int64), c.view(np.int64))


def test_interval_sign_partition_host_buffers_and_errors(cuda_device):
    # host (pinned-staging) path through the partition, and the invalid-
    # interval status raised by the classifier
    wl = W.c5()
    prog = pe.compile(wl.poly, wl.schemes)
    prog.set_tuning(iv_partition_min=1)
    lo, hi = wl.points(300_000)
    ev = pe.Evaluator(pe.IntervalDomain(), prog)
    got = ev.evaluate((lo, hi))
    o = pyoracle.Oracle(wl.poly, wl.schemes).eval_interval([lo[0][:2000]], [hi[0][:2000]])
    for a, c in zip(got, o):
        assert np.array_equal(np.asarray(a)[:2000].view(np.int64), c.view(np.int64))
    bad_lo = lo[0].copy()
    bad_lo[12345] = hi[0][12345] + 1.0
    with pytest.raises(ValueError):
        ev.evaluate(([bad_lo], hi))


@pytest.mark.parametrize("scheme", ["direct", "horner", "estrin", "balanced"])
@pytest.mark.parametrize("mode", ["kernel", "vm", "strict_replay"])
def test_interval_int64_coefficients_above_2_53_bit_exact(scheme, mode, cuda_device):
    # int64 coefficients that are not doubles are injected as the one-ulp-
    # widened interval around the nearest double (reference from_integer,
    # numeric.cpp:17-26; stream.cpp inject / interval_coefficient). Checked
    # against the golden vectors generated by the unmodified reference and
    # the oracle, through the specialised kernel (fast path + sign split),
    # the walk VM and the bit-level strict replay.
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "wide_int64_interval.npz"))
    p = pe.Polynomial(z["exponents"], z["coefficients"])
    assert p.coefficients.dtype == np.int64 and np.any(np.abs(p.coefficients.astype(object)) > 2**53)
    lo, hi = z["lo0"], z["hi0"]
    prog = pe.compile(p, pe.builtin_scheme(scheme))
    prog.set_tuning(**{"kernel": dict(jit_mode=1, iv_partition_min=1), "vm": dict(jit_mode=2),
                       "strict_replay": dict(jit_mode=1, iv_fast=-1)}[mode])
    glo, ghi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate(([_t(lo, cuda_device)], [_t(hi, cuda_device)]))
    glo, ghi = glo.cpu().numpy(), ghi.cpu().numpy()
    assert np.array_equal(glo.view(np.int64), z[f"out_lo_{scheme}"].view(np.int64))
    assert np.array_equal(ghi.view(np.int64), z[f"out_hi_{scheme}"].view(np.int64))
    olo, ohi = pyoracle.Oracle(p, [pe.builtin_scheme(scheme)]).eval_interval([lo], [hi])
    assert np.array_equal(glo.view(np.int64), olo.view(np.int64))
    assert np.array_equal(ghi.view(np.int64), ohi.view(np.int64))


@pytest.mark.parametrize("nvars", [1, 2])
@pytest.mark.parametrize("scheme", ["horner", "estrin", "balanced"])
def test_interval_fast_path_power_underflow_bit_exact(nvars, scheme, cuda_device):
    # Powers of tiny coordinates underflow: RN gives a zero endpoint and the
    # outward nextafter carries it across zero, so x^k straddles although x
    # does not (and although "squares are positive"). The fast path must send
    # such points to the exact replay instead of trusting the static sign
    # (found by scripts/fuzz_gpu.py seed 410119: results narrower than the
    # reference's). Unpartitioned and partitioned kernels, 1 and 2 variables.
    rng = np.random.default_rng(410119 + nvars)
    n = 2048
    if nvars == 1:
        ex = np.array([[29], [14], [7], [2], [1], [0]])
    else:
        ex = np.array([[29, 3], [14, 26], [6, 0], [2, 2], [1, 5], [0, 0]])
    p = pe.Polynomial(ex, rng.normal(size=len(ex)))
    x = rng.choice([-1.0, 1.0], n) * 10.0 ** rng.uniform(-320, 2, n)   # down to subnormals
    w = np.abs(x) * 10.0 ** rng.uniform(-17, 0, n) * (rng.random(n) < 0.7)
    lo, hi = [x.copy()], [x + w]
    if nvars == 2:
        y = rng.choice([-1.0, 1.0], n) * 10.0 ** rng.uniform(-3, 9, n)
        lo.append(y.copy())
        hi.append(y + np.abs(y) * 1e-9)
    sch = [pe.builtin_scheme(scheme)] * nvars
    olo, ohi = pyoracle.Oracle(p, sch).eval_interval(lo, hi)
    for tune in (dict(jit_mode=1), dict(jit_mode=1, iv_partition=-1),
                 dict(jit_mode=1, iv_partition_min=1), dict(jit_mode=1, iv_partition=3, iv_partition_min=1)):
        prog = pe.compile(p, sch)
        prog.set_tuning(**tune)
        glo, ghi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate(
            ([_t(a, cuda_device) for a in lo], [_t(a, cuda_device) for a in hi]))
        assert np.array_equal(glo.cpu().numpy().view(np.int64), olo.view(np.int64)), tune
        assert np.array_equal(ghi.cpu().numpy().view(np.int64), ohi.view(np.int64)), tune
