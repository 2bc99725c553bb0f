"""Seeded synthetic workloads for the five BASELINE.json configs.

No public dataset is involved: the reference names none. Every draw comes from
a pinned PCG64 stream per config through explicit transforms (stable across
numpy versions, unlike distribution helpers):
  U[-1,1]  : (int64(raw >> 11) - 2^52) * 2^-52
  N(0,1)   : Box-Muller on two U(0,1] draws built the same way
  int U[a,b]: raw % (b - a + 1) + a   (bias < 2^-60, irrelevant here)

C1  Hörner dense d1000 fp64, 1e5 points U[-1,1]           (CPU-runnable oracle)
C2  dense d1000 and d1023 fp64, Estrin vs balanced, 1e7 points
C3  bivariate total degree 40 (861 terms) int64 coeffs in [-8,8]\\{0},
    int64 points in [-2,2]^2, Hörner per variable, 1e7 points, bit-exact
C4  trivariate sparse 10,000 distinct terms, exponents 0..50 each, N(0,1)
    coeffs, balanced x3, 1e8 points U[-1,1]^3
C5  dense d200 fp64, Estrin, interval arithmetic, 1e8 intervals [x, x+1e-6]
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .api import BuiltinScheme, FunctionScheme, Polynomial

SEED_BASE = 13075655


def _rng(tag: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + tag))


def uniform_pm1(rng: np.random.Generator, n: int) -> np.ndarray:
    raw = rng.bit_generator.random_raw(n).astype(np.uint64)
    return ((raw >> np.uint64(11)).astype(np.int64) - (1 << 52)).astype(np.float64) * 2.0**-52


def uniform_01_open(rng: np.random.Generator, n: int) -> np.ndarray:
    raw = rng.bit_generator.random_raw(n).astype(np.uint64)
    return ((raw >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0**-53


def normal(rng: np.random.Generator, n: int) -> np.ndarray:
    u1 = uniform_01_open(rng, n)
    u2 = uniform_01_open(rng, n)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def uniform_int(rng: np.random.Generator, n: int, lo: int, hi: int) -> np.ndarray:
    raw = rng.bit_generator.random_raw(n).astype(np.uint64)
    return (raw % np.uint64(hi - lo + 1)).astype(np.int64) + lo


@dataclass
class Workload:
    name: str
    poly: Polynomial
    schemes: list
    domain: str            # "f64" | "i64" | "interval"
    n_points: int
    tag: int
    note: str = ""
    extra: dict = field(default_factory=dict)

    def points(self, n: int | None = None, offset_tag: int = 0):
        """SoA coordinates (list of arrays); intervals: (lo_list, hi_list)."""
        n = self.n_points if n is None else n
        rng = _rng(1000 + self.tag + offset_tag)
        nv = self.poly.nvars
        if self.domain == "i64":
            return [uniform_int(rng, n, -2, 2) for _ in range(nv)]
        if self.domain == "interval":
            lo = [uniform_pm1(rng, n) for _ in range(nv)]
            hi = [x + 1e-6 for x in lo]  # RN fp64 add
            return lo, hi
        return [uniform_pm1(rng, n) for _ in range(nv)]


def dense_univariate(degree: int, rng) -> Polynomial:
    c = uniform_pm1(rng, degree + 1)
    return Polynomial(np.arange(degree, -1, -1, dtype=np.uint32).reshape(-1, 1), c, ("x",))


def c1() -> Workload:
    return Workload("C1_horner_d1000", dense_univariate(1000, _rng(1)),
                    [FunctionScheme(BuiltinScheme.horner)], "f64", 100_000, 1,
                    "Horner dense d1000 fp64, 1e5 points")


def c2(degree: int = 1000, scheme: str = "estrin") -> Workload:
    tag = 2 if degree == 1000 else 3
    return Workload(f"C2_{scheme}_d{degree}", dense_univariate(degree, _rng(tag)),
                    [FunctionScheme(BuiltinScheme[scheme])], "f64", 10_000_000, tag,
                    f"{scheme} dense d{degree} fp64, 1e7 points")


def c2_all() -> list:
    return [c2(d, s) for d in (1000, 1023) for s in ("estrin", "balanced")]


def c3() -> Workload:
    rng = _rng(4)
    exps, coefs = [], []
    for i in range(41):
        for j in range(41 - i):
            exps.append((i, j))
    c = uniform_int(rng, len(exps), -8, 8)
    while (c == 0).any():  # resample zeros (reference bench.cpp:119)
        z = c == 0
        c[z] = uniform_int(rng, int(z.sum()), -8, 8)
    coefs = c
    poly = Polynomial(np.array(exps, dtype=np.uint32), coefs.astype(np.int64), ("x", "y"))
    return Workload("C3_bivariate_td40_i64", poly,
                    [FunctionScheme(BuiltinScheme.horner)] * 2, "i64", 10_000_000, 4,
                    "bivariate total degree 40, int64, Horner/Horner, 1e7 points")


def c4(n_terms: int = 10_000) -> Workload:
    rng = _rng(5)
    seen, exps = set(), []
    while len(exps) < n_terms:
        e = tuple(int(v) for v in uniform_int(rng, 3, 0, 50))
        if e in seen:
            continue  # rejection dedup
        seen.add(e)
        exps.append(e)
    coefs = normal(rng, n_terms)
    poly = Polynomial(np.array(exps, dtype=np.uint32), coefs, ("x", "y", "z"))
    return Workload("C4_trivariate_sparse10k", poly,
                    [FunctionScheme(BuiltinScheme.balanced)] * 3, "f64", 100_000_000, 5,
                    "trivariate sparse 10k terms, balanced x3, 1e8 points")


def c5() -> Workload:
    return Workload("C5_interval_estrin_d200", dense_univariate(200, _rng(6)),
                    [FunctionScheme(BuiltinScheme.estrin)], "interval", 100_000_000, 6,
                    "Estrin dense d200, interval, 1e8 intervals [x, x+1e-6]")


ALL = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def fig1(degree: int, coeff_bits: int = 64, point_bits: int = 64, n_points: int = 64,
         seed: int = 0):
    """The paper's Figure-1 workload (reference bench.cpp:59-187 run_grid):
    dense degree-d polynomial, coefficients uniform in [1, 2^coeff_bits)
    (zero redrawn), points with exactly point_bits bits (top bit set).
    Returns (exponents, coefficients as Python ints, points as Python ints).
    Seeded PCG64 words through explicit transforms, like every config here."""
    rng = _rng(7000 + 131 * degree + seed)

    def rand_bits(bits):
        words = (bits + 63) // 64
        raw = rng.bit_generator.random_raw(words).astype(np.uint64)
        v = 0
        for w in raw[::-1]:
            v = (v << 64) | int(w)
        return v & ((1 << bits) - 1)

    coefs = []
    for _ in range(degree + 1):
        c = rand_bits(coeff_bits)
        while c == 0:
            c = rand_bits(coeff_bits)
        coefs.append(c)
    exps = list(range(degree, -1, -1))
    points = [rand_bits(point_bits - 1) + (1 << (point_bits - 1)) for _ in range(n_points)]
    return exps, coefs, points
