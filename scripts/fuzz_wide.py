"""Randomised parity sweep of the wide-integer walk (pe_eval_wide) against the
unmodified reference BigInt, word for word: random uni- / multivariate
polynomials, signed coefficients and points of random bit sizes (zero,
powers of two and all-ones limbs mixed in), random scheme combinations,
batch sizes and CTA shapes (one warp / several warps per point).
Also cross-checks small cases against Python integer arithmetic.

  python scripts/fuzz_wide.py [seconds] [first_seed]
"""
import json
import os
import sys
import time
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
import pyoracle  # noqa: E402


def big(rng, bits, signed=True):
    kind = rng.integers(0, 10)
    if kind == 0:
        v = 0
    elif kind == 1:
        v = 1 << int(rng.integers(0, bits + 1))        # power of two: zero limbs below
    elif kind == 2:
        v = (1 << int(rng.integers(1, bits + 1))) - 1  # all-ones limbs
    else:
        b = int(rng.integers(1, bits + 1))
        v = int.from_bytes(rng.bytes((b + 7) // 8), "little") >> ((-b) % 8)
    return -v if signed and rng.random() < 0.5 else v


def scheme(rng):
    up, lo = (pe.BuiltinScheme(int(v)) for v in rng.integers(0, 4, 2))
    return pe.FunctionScheme(up, lo, int(rng.choice([0, 0, 1, 2, 5, 16])))


def check(seed):
    rng = np.random.default_rng(seed)
    nv = int(rng.choice([1, 1, 1, 2, 3]))
    if nv == 1:
        d = int(rng.choice([rng.integers(0, 12), rng.integers(12, 80), rng.integers(80, 200)]))
        ex = np.arange(d, -1, -1) if rng.random() < 0.6 else np.unique(rng.integers(0, d + 1, d // 3 + 1))
        ex = ex.reshape(-1, 1)
    else:
        ex = np.unique(rng.integers(0, int(rng.choice([3, 6, 10])), size=(int(rng.integers(1, 60)), nv)), axis=0)
    cbits = int(rng.choice([8, 64, 65, 200, 700, 2048]))
    pbits = int(rng.choice([3, 64, 65, 130, 600, 2048]))
    if len(ex) * max(1, int(ex.max())) * pbits > 6_000_000:  # keep results below ~100k limbs
        pbits = 64
    coefs = [big(rng, cbits) or 1 for _ in range(len(ex))]
    n = int(rng.choice([1, 3, 33, 150]))
    pts = [[big(rng, pbits) for _ in range(n)] for _ in range(nv)]
    sch = [scheme(rng) for _ in range(nv)]
    prog = pe.compile_wide(ex.tolist(), coefs, sch)
    block = int(rng.choice([0, 32, 64, 128, 256]))
    if block:
        prog.set_tuning(block=block)
    L = max(pe.limbs_for(p) for p in pts)
    cols = [pe.ints_to_words(p, L) for p in pts]
    got = pe.evaluate_wide(prog, cols, as_words=True)
    ref = pyoracle.ReferenceWide(ex.tolist(), pe.ints_to_words(coefs, pe.limbs_for(coefs)), sch)
    bad = ref.mismatches(cols, got)
    assert bad == 0, f"{bad} of {n} points differ (block {block}, cbits {cbits}, pbits {pbits}, nv {nv})"
    if n <= 3:  # and against Python's own integers
        ints = pe.words_to_ints(got)
        for i in range(n):
            want = 0
            for c, e in zip(coefs, ex):
                t = c
                for v in range(nv):
                    t *= int(pts[v][i]) ** int(e[v])
                want += t
            assert ints[i] == want, "python integer cross-check"
    return block


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 700000
    t0 = time.time()
    cases, failures, blocks = 0, [], {}
    while time.time() - t0 < budget:
        print(f"seed {seed} t={time.time() - t0:.1f}", file=sys.stderr, flush=True)
        try:
            b = check(seed)
            blocks[b] = blocks.get(b, 0) + 1
        except Exception as e:  # noqa: BLE001
            failures.append({"seed": seed, "error": repr(e)[:300],
                             "where": traceback.format_exc().splitlines()[-2][:200]})
        cases += 1
        seed += 1
    print(json.dumps({"cases": cases, "by_block": blocks, "failures": failures,
                      "seconds": round(time.time() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()
