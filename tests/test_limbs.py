"""K-limb exact integer kernels (pe_eval_limbs): codegen and host logic."""
import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W


def test_limbs_needed_follows_the_bound():
    wl = W.c3()  # 861 terms, |c| <= 8, total degree 40
    prog = pe.compile(wl.poly, wl.schemes)
    assert prog.limbs_needed([2, 2]) == 1        # the C3 range fits int64
    assert prog.limbs_needed([4, 4]) == 2        # ~2^93
    assert prog.limbs_needed([1000, 1000]) == 7  # ~2^412
    assert prog.limbs_needed([2**40, 2**40]) == 0  # > 511 bits


@pytest.mark.parametrize("k", [1, 3])
def test_limb_kernels_compile(k):
    wl = W.c3()
    prog = pe.compile(wl.poly, wl.schemes)
    ptx = prog.ptx(pe.DOMAIN_LIMBS(k))
    assert ptx.count(".param .u64 pe_out") == k
    if k >= 3:
        assert "madc.hi.u64" in ptx and "addc.cc.u64" in ptx
    assert prog.compile_only(pe.DOMAIN_LIMBS(k)) > 0


def test_limb_arguments_validated():
    wl = W.c3()
    prog = pe.compile(wl.poly, wl.schemes)
    ev = pe.Evaluator(pe.BigIntDomain(), prog)
    x = [np.zeros(4, np.int64)] * 2
    for k in (0, 9):
        with pytest.raises(ValueError):
            ev.evaluate_limbs(x, limbs=k)
    fp = pe.compile(W.c2(1000, "estrin").poly, W.c2(1000, "estrin").schemes)
    with pytest.raises(ValueError):
        fp.limbs_needed([1])


def test_limbs_to_int_twos_complement():
    vals = [0, 1, -1, 2**64 - 1, -(2**64), 2**100 + 12345, -(2**126) + 7]
    k = 2
    limbs = [np.array([(v % (1 << 128)) >> (64 * j) & ((1 << 64) - 1) for v in vals],
                      dtype=np.uint64) for j in range(k)]
    assert list(pe.limbs_to_int(limbs)) == vals
