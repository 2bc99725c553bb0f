"""Lowering + PTX emission + in-process ptxas (no GPU needed).

Checks that every config's specialised kernel compiles for sm_100a in every
applicable domain, and that the fused fp64 stream issues exactly the
algorithmic work F of SURVEY §8d (one DFMA per powered record + the power
table), i.e. every add of the reference walk was fused or folded.
"""
import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W

CASES = {
    "c1": W.c1, "c2e1000": lambda: W.c2(1000, "estrin"), "c2b1000": lambda: W.c2(1000, "balanced"),
    "c2e1023": lambda: W.c2(1023, "estrin"), "c3": W.c3, "c4": W.c4, "c5": W.c5,
}


@pytest.mark.parametrize("name", list(CASES))
def test_kernels_compile_for_sm100a(name):
    wl = CASES[name]()
    prog = pe.compile(wl.poly, wl.schemes)
    if wl.domain == "i64":
        doms = [pe.DOMAIN_I64, pe.DOMAIN_I64F]
    elif wl.domain == "interval":
        doms = [pe.DOMAIN_INTERVAL, pe.DOMAIN_F64]
    else:
        doms = [pe.DOMAIN_F64] + ([pe.DOMAIN_F64_STRICT] if name != "c4" else [])
    for d in doms:
        assert prog.compile_only(d) > 1000
        ptx = prog.ptx(d)
        assert ".target sm_100a" in ptx


@pytest.mark.parametrize("name", ["c1", "c2e1000", "c2b1000", "c2e1023", "c4"])
def test_fused_fp64_issues_exactly_F(name):
    # one sectioned kernel: F exactly; sections after the first rebuild only
    # the powers they read (C4: 4 sections, +184 multiplies = 1.5 %)
    wl = CASES[name]()
    prog = pe.compile(wl.poly, wl.schemes)
    prog.set_tuning(section_ops=2**32 - 1)
    inf = prog.info()
    F = inf["walk_muls"] + inf["power_muls"]
    assert prog.kernel_stats(pe.DOMAIN_F64)["fp_ops"] == F
    prog.set_tuning()
    k = prog.f64_slices()
    fp = prog.kernel_stats(pe.DOMAIN_F64)["fp_ops"]
    assert F <= fp <= F + (k - 1) * inf["power_muls"]
    assert (k > 1) == (name == "c4")
    if k > 1:
        ptx = prog.ptx(pe.DOMAIN_F64)
        assert ptx.count("bar.sync 0;") >= k and ptx.count(".func pe_section") == k


def test_sections_are_functions_over_tile_groups():
    # C4: one persistent kernel calling one function per section; every
    # section loads the 3 coordinates of its tile, the live values cross the
    # cuts through the scratch slot (as many loads as stores), and the
    # module compiles
    wl = W.c4()
    prog = pe.compile(wl.poly, wl.schemes)
    ptx = prog.ptx(pe.DOMAIN_F64)
    k = prog.f64_slices()
    assert k >= 3
    assert ptx.count("call.uni pe_section") == k
    assert ptx.count("ld.global.nc.f64 %x") == 3 * k
    assert ptx.count("ld.global.f64 %v") == ptx.count("st.global.f64 [%ga]") > 0
    # the shared-memory coefficient tier arrives by one TMA bulk copy per CTA
    assert "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes" in ptx
    assert prog.compile_only(pe.DOMAIN_F64) > 0


def test_int64_fused_issues_one_mad_per_record():
    wl = W.c3()
    prog = pe.compile(wl.poly, wl.schemes)
    inf = prog.info()
    assert prog.kernel_stats(pe.DOMAIN_I64)["int_ops"] == inf["walk_muls"] + inf["power_muls"]


def test_strict_fp64_replays_reference_op_counts():
    wl = W.c2(1000, "balanced")
    prog = pe.compile(wl.poly, wl.schemes)
    inf = prog.info()
    # strict = the reference sequence: every walk add and mul + power table
    assert prog.kernel_stats(pe.DOMAIN_F64_STRICT)["fp_ops"] == \
        inf["walk_adds"] + inf["walk_muls"] + inf["power_muls"]


def test_i64_domain_rejects_fp_coefficients():
    wl = W.c2(1000, "estrin")
    prog = pe.compile(wl.poly, wl.schemes)
    with pytest.raises(ValueError):
        prog.kernel_stats(pe.DOMAIN_I64)


def test_coefficient_tiers_large_program():
    # > 8000 distinct coefficient words spill from the constant bank into the
    # parameter tier and then global memory; the kernel must still build
    rng = np.random.default_rng(11)
    n = 12_100
    p = pe.Polynomial(np.arange(n - 1, -1, -1).reshape(-1, 1), rng.uniform(-1, 1, n))
    prog = pe.compile(p, pe.builtin_scheme("estrin"))
    prog.set_tuning(lanes=1, section_ops=2**32 - 1)  # one plain kernel, short ptxas run
    ptx = prog.ptx(pe.DOMAIN_F64)
    assert "pe_pcoef" in ptx and "ld.global.nc.f64 %c" in ptx
    assert prog.compile_only(pe.DOMAIN_F64) > 0
    # sectioned: section functions cannot read kernel parameters; the
    # overflow beyond the constant bank goes to shared memory
    prog.set_tuning(lanes=1)
    ptx = prog.ptx(pe.DOMAIN_F64)
    assert "pe_pcoef" not in ptx and "ld.shared" in ptx and prog.f64_slices() > 1
    assert prog.compile_only(pe.DOMAIN_F64) > 0


def test_horner_chain_becomes_counted_loop():
    # C1: one 999-step fma(acc, x, c) chain -> a loop over a constant-bank
    # array (same FMA sequence, so results are bit-identical; see
    # test_gpu_edges)
    wl = W.c1()
    prog = pe.compile(wl.poly, wl.schemes)
    ptx = prog.ptx(pe.DOMAIN_F64)
    assert ptx.count("bra.uni $Lrun") == 1
    assert ".const .align 16 .b64 pe_run0[1015]" in ptx  # 999 words + 2 trips of padding
    assert prog.kernel_stats(pe.DOMAIN_F64)["fp_ops"] == 1000
    assert prog.compile_only(pe.DOMAIN_F64) > 0
    prog2 = pe.compile(wl.poly, wl.schemes)
    prog2.set_tuning(chain_min=2**32 - 1)
    assert "$Lrun" not in prog2.ptx(pe.DOMAIN_F64)
    assert prog2.kernel_stats(pe.DOMAIN_F64)["fp_ops"] == 1000


def test_chain_loops_int64_domains():
    rng = np.random.default_rng(5)
    d = 150
    p = pe.Polynomial(np.arange(d, -1, -1).reshape(-1, 1),
                      rng.integers(1, 9, d + 1).astype(np.int64))
    prog = pe.compile(p, pe.builtin_scheme("horner"))
    for dom in (pe.DOMAIN_I64, pe.DOMAIN_I64F):
        ptx = prog.ptx(dom)
        assert "$Lrun0:" in ptx
        assert prog.compile_only(dom) > 0


def test_sparse_horner_splits_runs_at_gaps():
    # a gap changes the multiplier (x -> x^k): runs stop there
    e = np.array([300, 299, 298] + list(range(200, -1, -1))).reshape(-1, 1)
    c = np.linspace(0.5, 1.5, len(e))
    prog = pe.compile(pe.Polynomial(e, c), pe.builtin_scheme("horner"))
    ptx = prog.ptx(pe.DOMAIN_F64)
    assert ptx.count("bra.uni $Lrun") == 1  # the 200-long dense tail
    assert prog.compile_only(pe.DOMAIN_F64) > 0


def _kernel_words(ptx):
    """Every 64-bit coefficient word a kernel can read: the constant-bank
    array, the parameter tier is absent at these sizes, plus immediates."""
    import re
    words = set()
    for m in re.finditer(r"\.const \.align \d+ \.b64 pe_coef\[\d+\] = \{([^}]*)\}", ptx, re.S):
        words |= {int(w, 16) for w in re.findall(r"0x[0-9A-Fa-f]{16}", m.group(1))}
    words |= {int(w, 16) for w in re.findall(r"mov\.b64 %c\d+, (0x[0-9A-Fa-f]{16});", ptx)}
    return words


@pytest.mark.parametrize("domain", ["f64", "f64strict", "i64", "i64f"])
def test_coefficient_words_in_domain_format(domain):
    # The reference worked example (eval_test.cpp:80-93) with int64
    # coefficients; through both coefficient regions (uniform-bound words and
    # the register-bound second region), the kernel reads each coefficient in
    # the domain's own word format: doubles for the FP64 kernels, raw
    # integers for the int64 kernel.
    import struct
    e, c = [8, 7, 6, 5, 4, 3, 2, 1, 0], [3, -1, 2, 1, -4, 9, -3, -2, 1]
    d = {"f64": pe.DOMAIN_F64, "f64strict": pe.DOMAIN_F64_STRICT, "i64": pe.DOMAIN_I64,
         "i64f": pe.DOMAIN_I64F}[domain]
    p = pe.Polynomial(np.array(e).reshape(-1, 1), np.array(c, dtype=np.int64))
    for scheme in ("direct", "horner", "estrin", "balanced"):
        ptx = pe.compile(p, pe.builtin_scheme(scheme)).ptx(d)
        if domain == "i64":
            want = {v & (2**64 - 1) for v in c}
        else:
            want = {struct.unpack("<Q", struct.pack("<d", float(v)))[0] for v in c}
        got = _kernel_words(ptx) - {0}
        assert want <= got, (scheme, sorted(want - got))
        assert got <= want, (scheme, sorted(got - want))


def test_interval_fixup_entry_has_finite_case_replay():
    # The fixup replays a listed point with the finite-case primitives first
    # (directed-rounding nextafter, plain products + scan-order min/max,
    # NaN-poisoned accumulator) and keeps the bit-level replay behind the
    # %pmid branch. The replay is a function of the point index; the entry
    # strides over the list and calls it per point (inside a loop ptxas
    # would hoist and spill the replay's coefficient loads).
    wl = W.c5()
    prog = pe.compile(wl.poly, wl.schemes)
    ptx = prog.ptx(pe.DOMAIN_INTERVAL)
    fn = ptx[ptx.index(".func pe_fix_point"):ptx.index(".visible .entry")]
    assert "%macc" in fn and "@%pmid bra $Lexact" in fn
    assert "sub.rm.f64" in fn and "add.rn.f64 %tf" in fn
    fix = ptx[ptx.index(".entry pe_walk_interval_fix"):]
    assert "call.uni pe_fix_point" in fix and "bra $Lfix" in fix
    prog.set_tuning(iv_mid=-1)
    ptx0 = prog.ptx(pe.DOMAIN_INTERVAL)
    assert prog.compile_only(pe.DOMAIN_INTERVAL) > 0
    assert "%macc" not in ptx0


@pytest.mark.parametrize("name", ["c2e1000", "c3", "c4"])
def test_list_scheduler_keeps_ops_and_words(name):
    # The latency-aware reordering (on by default for wide programs like C4,
    # sched_window forces it elsewhere) only permutes SSA ops: the kernel
    # issues the same FP64 work and reads the same coefficient words.
    wl = CASES[name]()
    dom = pe.DOMAIN_I64F if wl.domain == "i64" else pe.DOMAIN_F64
    plain = pe.compile(wl.poly, wl.schemes)
    plain.set_tuning(sched_window=1)
    a, fa = plain.ptx(dom), plain.kernel_stats(dom)["fp_ops"]
    sched = pe.compile(wl.poly, wl.schemes)
    sched.set_tuning(sched_window=32, sched_distance=6)
    b, fb = sched.ptx(dom), sched.kernel_stats(dom)["fp_ops"]
    assert a != b
    assert fa == fb
    if name != "c4":  # (C4's 10k words overflow the constant bank: only part is in the text)
        assert _kernel_words(a) - {0} == _kernel_words(b) - {0}  # (section padding words)
    for op in ("fma.rn.f64", "mul.rn.f64", "add.rn.f64"):
        assert a.count(op) == b.count(op), op


def test_cubin_cache_survives_corruption_and_concurrency(tmp_path, monkeypatch):
    # the on-disk cubin cache: entries carry a length + checksum header and
    # are published by rename from a per-writer temporary, so concurrent
    # compiles of one PTX and a truncated entry both end in a valid cubin
    from concurrent.futures import ThreadPoolExecutor
    monkeypatch.setenv("PE_CACHE_DIR", str(tmp_path))
    wl = W.c2(1000, "estrin")

    def build(_):
        return pe.compile(wl.poly, wl.schemes).compile_only(pe.DOMAIN_F64)

    with ThreadPoolExecutor(4) as ex:
        sizes = list(ex.map(build, range(4)))
    assert len(set(sizes)) == 1 and sizes[0] > 0
    files = [f for f in tmp_path.iterdir() if f.suffix == ".cubin"]
    assert len(files) == 1 and not [f for f in tmp_path.iterdir() if ".tmp" in f.name]
    files[0].write_bytes(files[0].read_bytes()[:100])  # truncated entry
    assert build(0) == sizes[0]
    assert files[0].stat().st_size > 1000  # rewritten


def test_sectioned_kernel_with_all_coefficient_tiers_compiles():
    # 20k distinct coefficients: constant bank, the shared-memory tier up to
    # the 48 KB static limit (with the TMA mbarrier), global beyond
    rng = np.random.default_rng(12)
    d = 20_000
    p = pe.Polynomial(np.arange(d, -1, -1).reshape(-1, 1), rng.uniform(-1, 1, d + 1))
    prog = pe.compile(p, pe.builtin_scheme("estrin"))
    assert prog.f64_slices() > 1
    ptx = prog.ptx(pe.DOMAIN_F64)
    assert "ld.shared" in ptx and "ld.global.nc.f64 %c" in ptx
    assert prog.compile_only(pe.DOMAIN_F64) > 0


def test_interval_injection_of_int64_coefficients_above_2_53():
    # reference from_integer (numeric.cpp:17-26): an int64 coefficient that is
    # not a double becomes [next_down(RN(c)), next_up(RN(c))]; exact ones a
    # point interval. The words are baked into the constant bank.
    import struct

    def word(d):
        return "0x%016X" % struct.unpack("<Q", struct.pack("<d", d))[0]

    c = 2**53 + 1
    p = pe.Polynomial(np.array([[1], [0]]), np.array([c, 5], dtype=np.int64))
    ptx = pe.compile(p, pe.builtin_scheme("horner")).ptx(pe.DOMAIN_INTERVAL)
    near = float(c)  # RN-even: 2^53
    assert near == 2.0**53
    assert f"{word(np.nextafter(near, -np.inf))}, {word(np.nextafter(near, np.inf))}" in ptx
    assert word(5.0) in ptx
    # exactly representable large coefficient: no widening
    q = pe.Polynomial(np.array([[1], [0]]), np.array([2**60, 5], dtype=np.int64))
    ptx = pe.compile(q, pe.builtin_scheme("horner")).ptx(pe.DOMAIN_INTERVAL)
    assert word(2.0**60) in ptx and word(np.nextafter(2.0**60, np.inf)) not in ptx


def test_split_kernel_point_functions_are_divergence_safe():
    # The one-pass sign split calls the program's and the mirrored program's
    # point functions from threads of one CTA (and, in the boundary warp, of
    # one warp). Two hazards found on the GPU: a CTA barrier inside a point
    # function deadlocks the CTA, and .param arguments shared by two calls
    # bind only to the first call (the second reads stale registers).
    import re
    wl = W.c5()
    prog = pe.compile(wl.poly, wl.schemes)
    prog.set_tuning(iv_partition=3)
    ptx = prog.ptx(pe.DOMAIN_INTERVAL)
    assert "pe_walk_interval_split" in ptx
    for name in ("pe_iv_pos", "pe_iv_neg", "pe_fix_point"):
        start = ptx.index(".func")
        m = re.search(r"\.func[^\n]*\b%s\(" % name, ptx)
        assert m, name
        body = ptx[m.start():ptx.index("\n}\n", m.start())]
        assert "bar.sync" not in body, name
    # every call to a point function sits in its own scope with its own
    # st.param stores
    entry = ptx[ptx.index(".entry pe_walk_interval_split"):]
    entry = entry[:entry.index("\n}\n")]
    scopes = re.findall(r"\{\n(.*?)\n  \}", entry, flags=re.S)
    calls = [sc for sc in scopes if "call " in sc]
    assert len(calls) == 2
    for sc in calls:
        assert sc.count("call ") == 1 and sc.count("st.param.f64") == 2
