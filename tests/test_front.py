"""Host front-end parity (no GPU): schemes, trees, lazy heights, compile.

The product's native front-end (through the C ABI) is compared with the
reference's own known answers, with the committed DOT goldens, with the C
oracle, and — where /root/reference was compiled into oracle/_ref — with the
unmodified reference library itself.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import _lib as L
from paper_1307_5655_b200 import workloads as W
import pyoracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
EXAMPLE = ([8, 7, 6, 5, 4, 3, 2, 1, 0], [3, -1, 2, 1, -4, 9, -3, -2, 1])
SCHEMES = ["direct", "horner", "estrin", "balanced"]


def example(dtype=np.int64):
    e, c = EXAMPLE
    return pe.Polynomial(np.array(e).reshape(-1, 1), np.array(c, dtype=dtype))


# --------------------------------------------------------------- ABI surface

def test_header_symbols_all_exported():
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "polyeval_b200.h")).read()
    declared = set(re.findall(r"^\S.*?\b(pe_[a-z0-9_]+)\(", hdr, flags=re.M))
    assert "pe_eval_f64" in declared and "pe_program_create" in declared
    lib = L.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in L.EXPORTS}
    assert declared == bound, declared ^ bound


def test_version_string():
    assert b"sm_100a" in L.lib().pe_version()


# --------------------------------------------------------------- schemes

def test_scheme_split_values():
    # reference scheme_test.cpp:10-25
    assert pe.builtin_scheme("direct").split(5) == 5
    assert pe.builtin_scheme("horner").split(5) == 1
    es = pe.builtin_scheme("estrin")
    assert [es.split(k) for k in (7, 8, 9, 1)] == [4, 8, 8, 1]
    b = pe.builtin_scheme("balanced")
    assert [b.split(k) for k in (8, 1, 9)] == [4, 1, 5]  # D1: ceil(k/2)


def test_threshold_combine():
    # reference scheme_test.cpp:34-62
    c = pe.threshold_combine(pe.builtin_scheme("estrin"), pe.builtin_scheme("horner"), 10)
    assert (c.split(16), c.split(10), c.split(11)) == (16, 1, 8)
    assert c.name == "estrin:horner@10"
    c2 = pe.threshold_combine(pe.builtin_scheme("balanced"), pe.builtin_scheme("horner"), 2)
    assert (c2.split(3), c2.split(4)) == (2, 2)
    with pytest.raises(ValueError):
        pe.threshold_combine(pe.builtin_scheme("direct"), pe.builtin_scheme("horner"), 0)
    assert pe.scheme_from_name("balanced:horner@2") == c2
    with pytest.raises(ValueError):
        pe.scheme_from_name("balanced:horner@0")


# --------------------------------------------------------------- trees / DOT

@pytest.mark.parametrize("scheme", SCHEMES)
def test_dot_matches_golden(scheme):
    prog = pe.compile(example(), pe.builtin_scheme(scheme))
    golden = open(os.path.join(GOLDEN, f"ref_dot_{scheme}.dot")).read()
    assert prog.dot() == golden


@pytest.mark.parametrize("scheme", SCHEMES)
def test_golden_dot_is_the_reference_fixture(scheme):
    src = f"/root/reference/proj/tests/golden/example_{scheme}.dot"
    if not os.path.exists(src):
        pytest.skip("reference tree not present (GPU box)")
    assert open(src).read() == open(os.path.join(GOLDEN, f"ref_dot_{scheme}.dot")).read()


def test_estrin_max_lazy_height_is_two():
    # discrepancy D3: the code (and acceptance_test.cpp:114-116) pins 2
    prog = pe.compile(example(), pe.builtin_scheme("estrin"))
    assert prog.info()["register_count"] == 3


def test_compile_layouts():
    # reference eval_test.cpp:23-60
    single = pe.compile(pe.Polynomial(np.array([[3]]), np.array([7], dtype=np.int64)),
                        pe.builtin_scheme("balanced"))
    assert single.info()["records"] == 1 and single.info()["register_count"] == 1
    assert single.exponent_set(0) == [3]
    r = single.records()
    assert r[0].tolist() == [0, 0, -1, 0, 0]
    horner = pe.compile(example(), pe.builtin_scheme("horner"))
    assert horner.info()["register_count"] == 1
    assert horner.exponent_set(0) == [1]
    rec = horner.records()
    assert (rec[:-1, 2] >= 0).all() and rec[-1, 2] == -1 and rec[-1, 0] == -1
    direct = pe.compile(example(), pe.builtin_scheme("direct"))
    assert direct.info()["register_count"] == 2
    assert direct.exponent_set(0) == [1, 2, 3, 4, 5, 6, 7, 8]
    assert direct.info()["root_children"] == 8


def _random_poly(rng, max_degree=64, dense=None):
    d = int(rng.integers(0, max_degree + 1))
    if dense if dense is not None else rng.integers(0, 2):
        ex = list(range(d + 1))
    else:
        want = int(rng.integers(1, d + 2))
        ex = sorted(set([d] + list(rng.integers(0, d + 1, size=want))))
    c = rng.integers(-(2 ** 15), 2 ** 15, size=len(ex))
    c[c == 0] = 1
    return pe.Polynomial(np.array(ex).reshape(-1, 1), c.astype(np.int64))


def test_records_match_oracle_random():
    rng = np.random.default_rng(300)
    for _ in range(60):
        p = _random_poly(rng)
        for s in SCHEMES:
            sch = [pe.builtin_scheme(s)]
            prog = pe.compile(p, sch)
            rec, rc = pyoracle.Oracle(p, sch).records()
            assert np.array_equal(prog.records(), rec)
            assert prog.info()["register_count"] == rc
            # register_count <= bit_width(records) (eval_test.cpp:62-78)
            assert rc <= int(prog.info()["records"]).bit_length()


def test_op_count_identities():
    # eval_test.cpp:182-216: adds = (nodes-1) + #with_children, muls = #with_power
    rng = np.random.default_rng(303)
    for _ in range(25):
        p = _random_poly(rng)
        for s in SCHEMES:
            prog = pe.compile(p, pe.builtin_scheme(s))
            rec = prog.records()
            inf = prog.info()
            assert inf["walk_adds"] == (len(rec) - 1) + int(rec[:, 3].sum())
            assert inf["walk_muls"] == int((rec[:, 0] >= 0).sum())


def test_invalid_scheme_and_arity_errors():
    with pytest.raises(ValueError):
        pe.compile(example(), [pe.builtin_scheme("horner")] * 2)  # one scheme per variable
    with pytest.raises(ValueError):
        pe.Polynomial(np.array([[1, 2]]), np.array([1.0, 2.0]))  # coefficient count
    # non-finite fp64 coefficient is rejected at the boundary
    with pytest.raises(ValueError):
        pe.compile(pe.Polynomial(np.array([[1]]), np.array([np.inf])), pe.builtin_scheme("horner"))


def test_canonicalization_merges_and_drops():
    p = pe.Polynomial(np.array([[2], [2], [1], [0], [1]]), np.array([3, -3, 5, 1, -5], dtype=np.int64))
    prog = pe.compile(p, pe.builtin_scheme("balanced"))
    assert prog.info()["terms"] == 1  # only the constant 1 survives


@pytest.mark.skipif(not pyoracle.ref_available(), reason="reference library not built here")
@pytest.mark.parametrize("make", [W.c1, lambda: W.c2(1000, "estrin"), lambda: W.c2(1000, "balanced"),
                                  lambda: W.c2(1023, "estrin"), W.c3, W.c4, W.c5])
def test_compiled_program_matches_reference(make):
    wl = make()
    prog = pe.compile(wl.poly, wl.schemes)
    ref = pyoracle.Reference(wl.poly, wl.schemes)
    rr, rc = ref.records()
    assert np.array_equal(prog.records(), rr)
    assert prog.info()["register_count"] == rc
    for v in range(wl.poly.nvars):
        assert prog.exponent_set(v) == ref.exponent_set(v)


def test_survey_table_counts():
    # C2 estrin d1000 R=1001 muls 1000 adds 1500 regs 6; balanced
    # adds 1512; d1023 estrin == balanced trees (both 1535 adds); C5 adds 300.
    e = pe.compile(W.c2(1000, "estrin").poly, [pe.builtin_scheme("estrin")]).info()
    b = pe.compile(W.c2(1000, "balanced").poly, [pe.builtin_scheme("balanced")]).info()
    assert (e["records"], e["walk_muls"], e["walk_adds"], e["register_count"]) == (1001, 1000, 1500, 6)
    assert (b["walk_adds"], b["register_count"], b["exponent_set_sizes"][0]) == (1512, 6, 14)
    d1 = pe.compile(W.c2(1023, "estrin").poly, [pe.builtin_scheme("estrin")])
    d2 = pe.compile(W.c2(1023, "balanced").poly, [pe.builtin_scheme("balanced")])
    assert np.array_equal(d1.records(), d2.records()) and d1.info()["walk_adds"] == 1535
    c5 = pe.compile(W.c5().poly, W.c5().schemes).info()
    assert (c5["walk_adds"], c5["walk_muls"], c5["register_count"]) == (300, 200, 5)


def test_c_abi_error_contract():
    lib = L.lib()
    exps = (C.c_uint32 * 2)(1, 0)
    coefs = (C.c_double * 2)(1.0, 2.0)
    h = C.c_void_p()
    bad_scheme = (L.pe_scheme_desc * 1)(L.pe_scheme_desc(7, 0, 0))
    assert lib.pe_program_create(exps, coefs, 2, 1, bad_scheme, 0, C.byref(h)) == L.PE_EINVAL
    assert b"scheme" in lib.pe_last_error()
    ok = (L.pe_scheme_desc * 1)(L.pe_scheme_desc(3, 3, 0))
    assert lib.pe_program_create(exps, coefs, 2, 0, ok, 0, C.byref(h)) == L.PE_EINVAL  # nvars 0
    assert lib.pe_program_create(None, coefs, 2, 1, ok, 0, C.byref(h)) == L.PE_EINVAL
    assert lib.pe_program_create(exps, coefs, 2, 1, ok, 9, C.byref(h)) == L.PE_EINVAL  # coeff type
    assert lib.pe_program_create(exps, coefs, 2, 1, None, 0, C.byref(h)) == L.PE_EINVAL
    # zero terms is the zero polynomial, not an error
    assert lib.pe_program_create(None, None, 0, 1, ok, 0, C.byref(h)) == L.PE_OK
    lib.pe_program_destroy(h)
    # eval with n == 0 is a no-op; null program is EINVAL (no GPU needed)
    assert lib.pe_eval_f64(None, None, 0, None, None) == L.PE_EINVAL
    with pytest.raises(ValueError):
        pe.compile(pe.Polynomial(np.array([[1]]), np.array([1.0])), pe.FunctionScheme(
            pe.BuiltinScheme.estrin, pe.BuiltinScheme.horner, 0)).kernel_stats(9)


def test_scheme_range_violation_is_invalid_argument():
    # reference tree.cpp:41-44: a split outside (0, k] throws invalid_argument;
    # the builtins never do, so threshold on an out-of-range cutoff is the
    # only way through the ABI — every builtin combination must stay valid
    rng = np.random.default_rng(5)
    for up in range(4):
        for lo in range(4):
            for cut in (1, 2, 3, 7, 100):
                s = pe.FunctionScheme(pe.BuiltinScheme(up), pe.BuiltinScheme(lo), cut)
                p = _random_poly(rng, max_degree=40)
                rec, rc = pyoracle.Oracle(p, [s]).records()
                prog = pe.compile(p, [s])
                assert np.array_equal(prog.records(), rec) and prog.info()["register_count"] == rc


@pytest.mark.skipif(not pyoracle.ref_available(), reason="reference library not built here")
def test_multivariate_dot_matches_reference():
    # nested-coefficient labels render the inner polynomial over the suffix
    # variables (reference tree.cpp:290-309 + parser.cpp render)
    rng = np.random.default_rng(41)
    for nv in (2, 3):
        for trial in range(6):
            t = int(rng.integers(1, 40))
            ex = rng.integers(0, 6, size=(t, nv))
            c = rng.integers(-9, 10, size=t).astype(np.int64)
            c[c == 0] = 1
            p = pe.Polynomial(ex, c)
            for s in SCHEMES:
                sch = [pe.builtin_scheme(s)] * nv
                prog = pe.compile(p, sch)
                assert prog.dot() == pyoracle.Reference(p, sch).dot(), (nv, trial, s)
                rr, rc = pyoracle.Reference(p, sch).records()
                assert np.array_equal(prog.records(), rr) and prog.info()["register_count"] == rc


def test_deep_horner_builds_without_recursion():
    # the builder is iterative: a 200k-term Horner chain (tree depth 200k)
    # needs no deep stack
    n = 200_000
    p = pe.Polynomial(np.arange(n).reshape(-1, 1), np.ones(n, dtype=np.int64))
    prog = pe.compile(p, pe.builtin_scheme("horner"))
    inf = prog.info()
    assert inf["records"] == n and inf["register_count"] == 1 and inf["walk_muls"] == n - 1
