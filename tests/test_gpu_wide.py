"""GPU: arbitrary-width exact evaluation (pe_eval_wide, one CTA of 1-8 warps per point)
against the unmodified reference BigInt walk, word for word — the paper's
Figure-1 workload (reference bench.cpp run_grid defaults: 64-bit
coefficients and points; acceptance_test.cpp C09: 2048-bit at degrees
255 / 256) plus signed multivariate programs."""
import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W
import pyoracle

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not pyoracle.ref_available(), reason="oracle/_ref not built")]


# CTA sizes of the wide walk: one warp (narrow ops and the product assembly
# in registers, the shape of large batches), several warps (ranges of rows /
# blocks of columns per warp, the shape of small batches), the default
BLOCKS = [32, 128, 0]


def _check(exps, coefs, pts_per_var, schemes, device=None, block=0):
    prog = pe.compile_wide(exps, coefs, schemes)
    if block:
        prog.set_tuning(block=block)
    L = max(pe.limbs_for(p) for p in pts_per_var)
    cols = [pe.ints_to_words(p, L) for p in pts_per_var]
    got = pe.evaluate_wide(prog, cols, as_words=True)
    ref = pyoracle.ReferenceWide(exps, pe.ints_to_words(coefs, pe.limbs_for(coefs)),
                                 schemes if isinstance(schemes, list) else [schemes])
    assert ref.mismatches(cols, got) == 0
    return prog, cols, got


@pytest.mark.parametrize("degree", [0, 1, 7, 64, 255, 256])
@pytest.mark.parametrize("scheme", ["balanced", "estrin", "horner"])
@pytest.mark.parametrize("block", BLOCKS)
def test_fig1_grid_64bit(degree, scheme, block, cuda_device):
    exps, coefs, pts = W.fig1(degree, 64, 64, 37)
    _check(exps, coefs, [pts], pe.builtin_scheme(scheme), block=block)


@pytest.mark.parametrize("degree", [255, 256])
@pytest.mark.parametrize("scheme", ["balanced", "estrin"])
@pytest.mark.parametrize("block", BLOCKS)
def test_staircase_2048bit(degree, scheme, block, cuda_device):
    exps, coefs, pts = W.fig1(degree, 2048, 2048, 5)
    _check(exps, coefs, [pts], pe.builtin_scheme(scheme), block=block)


@pytest.mark.parametrize("block", BLOCKS)
def test_signed_multivariate(block, cuda_device):
    rng = np.random.default_rng(12)
    ex = np.unique(rng.integers(0, 9, size=(60, 3)), axis=0)
    coefs = [int(rng.integers(-(2**62), 2**62)) * (1 << int(rng.integers(0, 200))) for _ in range(len(ex))]
    pts = [[int(rng.integers(-(2**62), 2**62)) * (1 << int(rng.integers(0, 90))) for _ in range(33)]
           for _ in range(3)]
    pts[0][0], pts[1][0], pts[2][0] = 0, 0, 0
    pts[0][1] = -(2**150)
    _check(ex.tolist(), coefs, pts, [pe.builtin_scheme(s) for s in ("balanced", "estrin", "horner")],
           block=block)


@pytest.mark.parametrize("block", BLOCKS)
def test_signed_dense_wide_values(block, cuda_device):
    # negative coefficients and points of several hundred bits: negative
    # operands and products on the wide path (magnitudes, negated results,
    # carries that ripple across 32-limb rows: all-ones and zero limbs)
    rng = np.random.default_rng(77)
    d = 90
    coefs = [int(rng.integers(-(2**62), 2**62)) * (1 << int(rng.integers(0, 700))) - 1 for _ in range(d + 1)]
    coefs[3] = -(2**640)          # a power of two: zero limbs below the top
    coefs[5] = 2**704 - 1         # all-ones limbs
    pts = [int(rng.integers(-(2**62), 2**62)) * (1 << int(rng.integers(0, 300))) for _ in range(21)]
    pts[0], pts[1], pts[2], pts[3] = 0, -1, 1, -(2**320)
    exps = [[e] for e in range(d, -1, -1)]
    for scheme in ("balanced", "horner"):
        _check(exps, coefs, [pts], pe.builtin_scheme(scheme), block=block)


def test_python_ints_and_device_buffers_agree(cuda_device):
    import torch
    exps, coefs, pts = W.fig1(40, 192, 100, 11)
    prog = pe.compile_wide(exps, coefs, pe.builtin_scheme("balanced"))
    ints = pe.evaluate_wide(prog, [pts])
    assert ints == [sum(c * x ** e for c, e in zip(coefs, exps)) for x in pts]
    L = pe.limbs_for(pts)
    k = pe.wide_limbs(prog, L)
    dev_in = torch.from_numpy(pe.ints_to_words(pts, L).view(np.int64)).to(cuda_device)
    dev_out = torch.zeros((len(pts), k), dtype=torch.int64, device=cuda_device)
    import ctypes as C
    from paper_1307_5655_b200 import _lib as L_
    ptrs = (C.c_void_p * 1)(dev_in.data_ptr())
    ex = L_.pe_exec()
    ex.device = -1
    ex.synchronize = 1
    L_.check(L_.lib().pe_eval_wide(prog.handle, ptrs, L, len(pts), dev_out.data_ptr(), k, C.byref(ex)))
    assert pe.words_to_ints(dev_out.cpu().numpy().view(np.uint64)) == ints
