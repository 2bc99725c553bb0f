"""ORACLE / TEST INFRASTRUCTURE ONLY — ctypes access to the checkers.

  Oracle      the plain-C restatement (oracle/liboracle.so, pe_oracle.c)
  Reference   the unmodified reference library (oracle/_ref/libpolyeval_ref.so,
              compiled from /root/reference by oracle/Makefile), driven through
              its own compile()/Evaluator<D> API by ref_harness.cpp

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or the timed
CPU baseline — never as a product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpolyeval_ref.so")

DOM_DOUBLE, DOM_INTERVAL, DOM_INT64 = 0, 1, 2

_oracle = None
_ref = None


def _scheme_arrays(schemes):
    nv = len(schemes)
    up = (C.c_int * nv)(*[int(s.upper) for s in schemes])
    lo = (C.c_int * nv)(*[int(s.lower) for s in schemes])
    cut = (C.c_uint64 * nv)(*[int(s.cutoff) for s in schemes])
    return up, lo, cut


def _ptrs(arrays):
    return (C.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            raise ImportError(f"oracle not built: {ORACLE_SO} (make -C oracle)")
        lib = C.CDLL(ORACLE_SO)
        lib.oracle_create.restype = C.c_void_p
        lib.oracle_create.argtypes = [C.POINTER(C.c_uint32), C.c_void_p, C.c_size_t, C.c_uint32,
                                      C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_uint64), C.c_int]
        lib.oracle_destroy.argtypes = [C.c_void_p]
        lib.oracle_eval.restype = C.c_int
        lib.oracle_eval.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t,
                                    C.c_void_p, C.c_void_p]
        lib.oracle_abs_term_sum.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_double),
                                            C.c_size_t, C.c_uint32, C.c_void_p, C.c_size_t,
                                            C.POINTER(C.c_double)]
        lib.oracle_records.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_size_t,
                                       C.POINTER(C.c_size_t), C.POINTER(C.c_uint32)]
        lib.oracle_dot.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        lib.oracle_last_error.restype = C.c_char_p
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise ImportError(f"reference not built: {REF_SO} (make -C oracle ref)")
        lib = C.CDLL(REF_SO)
        lib.ref_create.restype = C.c_int
        lib.ref_create.argtypes = [C.POINTER(C.c_uint32), C.c_void_p, C.c_size_t, C.c_uint32,
                                   C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_uint64), C.c_int, C.POINTER(C.c_void_p)]
        lib.ref_destroy.argtypes = [C.c_void_p]
        lib.ref_dot.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        lib.ref_records.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_size_t,
                                    C.POINTER(C.c_size_t), C.POINTER(C.c_uint32)]
        lib.ref_exponents.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32), C.c_size_t,
                                      C.POINTER(C.c_size_t)]
        lib.ref_eval_f64.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int]
        lib.ref_eval_interval.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                          C.c_void_p, C.c_void_p, C.c_int]
        lib.ref_eval_i64.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int]
        lib.ref_eval_parallel_f64.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                              C.c_uint]
        lib.ref_time_parallel_interval.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                                   C.c_uint, C.POINTER(C.c_double)]
        lib.ref_time_parallel_i64.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint,
                                              C.POINTER(C.c_double)]
        lib.ref_export.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                   C.POINTER(C.c_size_t)]
        lib.ref_eval_limbs.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint32,
                                        C.c_void_p, C.c_int]
        lib.ref_create_wide.argtypes = [C.POINTER(C.c_uint32), C.c_void_p, C.c_uint32, C.c_size_t,
                                        C.c_uint32, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_void_p)]
        lib.ref_eval_wide_check.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_size_t,
                                            C.c_void_p, C.c_uint32, C.c_int, C.POINTER(C.c_size_t)]
        lib.ref_time_wide.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_size_t, C.c_int,
                                      C.POINTER(C.c_double)]
        lib.ref_last_error.restype = C.c_char_p
        _ref = lib
    return _ref


class Oracle:
    """C restatement of build -> lazy heights -> compile -> walk."""

    def __init__(self, poly, schemes):
        lib = oracle_lib()
        self.poly = poly
        self.integer = poly.coefficients.dtype == np.int64
        up, lo, cut = _scheme_arrays(schemes)
        self._keep = (poly.exponents, poly.coefficients)
        h = lib.oracle_create(poly.exponents.ctypes.data_as(C.POINTER(C.c_uint32)),
                              poly.coefficients.ctypes.data, poly.coefficients.shape[0],
                              poly.nvars, up, lo, cut, 1 if self.integer else 0)
        if not h:
            raise ValueError(lib.oracle_last_error().decode())
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            oracle_lib().oracle_destroy(self._h)
            self._h = None

    def eval_f64(self, coords):
        cols = [np.ascontiguousarray(c, dtype=np.float64) for c in coords]
        out = np.empty(cols[0].shape[0], dtype=np.float64)
        oracle_lib().oracle_eval(self._h, DOM_DOUBLE, _ptrs(cols), None, out.shape[0],
                                 out.ctypes.data, None)
        return out

    def eval_interval(self, lo, hi):
        lo = [np.ascontiguousarray(c, dtype=np.float64) for c in lo]
        hi = [np.ascontiguousarray(c, dtype=np.float64) for c in hi]
        n = lo[0].shape[0]
        olo, ohi = np.empty(n), np.empty(n)
        oracle_lib().oracle_eval(self._h, DOM_INTERVAL, _ptrs(lo), _ptrs(hi), n,
                                 olo.ctypes.data, ohi.ctypes.data)
        return olo, ohi

    def eval_i64(self, coords):
        cols = [np.ascontiguousarray(c, dtype=np.int64) for c in coords]
        out = np.empty(cols[0].shape[0], dtype=np.int64)
        st = oracle_lib().oracle_eval(self._h, DOM_INT64, _ptrs(cols), None, out.shape[0],
                                      out.ctypes.data, None)
        if st == 2:
            raise OverflowError("oracle: int64 overflow")
        return out

    def records(self):
        n, rc = C.c_size_t(), C.c_uint32()
        oracle_lib().oracle_records(self._h, None, 0, C.byref(n), C.byref(rc))
        buf = np.zeros(5 * max(1, n.value), dtype=np.int32)
        oracle_lib().oracle_records(self._h, buf.ctypes.data_as(C.POINTER(C.c_int32)), buf.size,
                                    C.byref(n), C.byref(rc))
        return buf[: 5 * n.value].reshape(-1, 5), rc.value

    def dot(self):
        n = C.c_size_t()
        if oracle_lib().oracle_dot(self._h, None, 0, C.byref(n)):
            raise ValueError("oracle_dot: nested trees not supported")
        buf = C.create_string_buffer(n.value + 1)
        oracle_lib().oracle_dot(self._h, buf, n.value + 1, C.byref(n))
        return buf.value.decode()


def abs_term_sum(poly, coords):
    """sum_t |c_t| prod_v |x_v|^a_tv per point (fp64 tolerance scale)."""
    cols = [np.ascontiguousarray(c, dtype=np.float64) for c in coords]
    coefs = np.ascontiguousarray(poly.coefficients, dtype=np.float64)
    out = np.empty(cols[0].shape[0])
    oracle_lib().oracle_abs_term_sum(poly.exponents.ctypes.data_as(C.POINTER(C.c_uint32)),
                                     coefs.ctypes.data_as(C.POINTER(C.c_double)), coefs.shape[0],
                                     poly.nvars, _ptrs(cols), out.shape[0],
                                     out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


class Reference:
    """The unmodified reference library through its own API (ref_harness.cpp)."""

    def __init__(self, poly, schemes):
        lib = ref_lib()
        self.integer = poly.coefficients.dtype == np.int64
        self.nvars = poly.nvars
        up, lo, cut = _scheme_arrays(schemes)
        h = C.c_void_p()
        self._keep = (poly.exponents, poly.coefficients)
        st = lib.ref_create(poly.exponents.ctypes.data_as(C.POINTER(C.c_uint32)),
                            poly.coefficients.ctypes.data, poly.coefficients.shape[0], poly.nvars,
                            up, lo, cut, 1 if self.integer else 0, C.byref(h))
        if st:
            raise ValueError(lib.ref_last_error().decode())
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                ref_lib().ref_destroy(self._h)
            except Exception:  # noqa: BLE001 — interpreter shutdown
                pass
            self._h = None

    def _check(self, st):
        if st:
            msg = ref_lib().ref_last_error().decode()
            if "int64" in msg:
                raise OverflowError(msg)
            raise ValueError(msg)

    def export(self):
        """The reference's own CompiledProgram, flattened (root first, nested
        programs pre-order) in the shape CompiledProgram.from_compiled takes,
        plus the per-variable exponent sets."""
        lib = ref_lib()
        nr, npg, ne = C.c_size_t(), C.c_size_t(), C.c_size_t()
        self._check(lib.ref_export(self._h, None, None, None, None, None, C.byref(nr),
                                   C.byref(npg), C.byref(ne)))
        f64 = np.zeros(nr.value, np.float64)
        i64 = np.zeros(nr.value, np.int64)
        ints = np.zeros((nr.value, 5), np.int32)
        info = np.zeros((npg.value, 6), np.uint32)
        ends = np.zeros(max(1, ne.value), np.uint32)
        self._check(lib.ref_export(self._h, f64.ctypes.data, i64.ctypes.data, ints.ctypes.data,
                                   info.ctypes.data, ends.ctypes.data, C.byref(nr), C.byref(npg),
                                   C.byref(ne)))
        programs = []
        for first, n, regs, var, e0, ne_k in info.tolist():
            recs = []
            for i in range(first, first + n):
                sub, ps, lazy, parent, reads = ints[i].tolist()
                recs.append({"coeff": int(i64[i]) if self.integer else float(f64[i]), "sub": sub,
                             "power_slot": ps, "lazy_slot": lazy, "parent_slot": parent,
                             "reads_register": bool(reads)})
            programs.append({"records": recs, "register_count": regs, "variable": var,
                             "root_child_ends": ends[e0:e0 + ne_k].tolist()})
        sets = [self.exponents(v) for v in range(self.nvars)]
        return programs, sets

    def exponents(self, v):
        lib = ref_lib()
        n = C.c_size_t()
        buf = (C.c_uint32 * 4096)()
        self._check(lib.ref_exponents(self._h, v, buf, 4096, C.byref(n)))
        if n.value > 4096:
            buf = (C.c_uint32 * n.value)()
            self._check(lib.ref_exponents(self._h, v, buf, n.value, C.byref(n)))
        return list(buf[:n.value])

    def eval_f64(self, coords, threads=1):
        cols = [np.ascontiguousarray(c, dtype=np.float64) for c in coords]
        out = np.empty(cols[0].shape[0])
        self._check(ref_lib().ref_eval_f64(self._h, _ptrs(cols), out.shape[0], out.ctypes.data,
                                           threads))
        return out

    def eval_parallel_f64(self, coords, workers):
        cols = [np.ascontiguousarray(c, dtype=np.float64) for c in coords]
        out = np.empty(cols[0].shape[0])
        self._check(ref_lib().ref_eval_parallel_f64(self._h, _ptrs(cols), out.shape[0],
                                                    out.ctypes.data, workers))
        return out

    def seconds_parallel_interval(self, lo, hi, workers):
        """Wall time of evaluate_parallel(workers) over the intervals (reference clock)."""
        lo = [np.ascontiguousarray(c, dtype=np.float64) for c in lo]
        hi = [np.ascontiguousarray(c, dtype=np.float64) for c in hi]
        sec = C.c_double()
        self._check(ref_lib().ref_time_parallel_interval(self._h, _ptrs(lo), _ptrs(hi), lo[0].shape[0],
                                                         workers, C.byref(sec)))
        return sec.value

    def seconds_parallel_i64(self, coords, workers):
        cols = [np.ascontiguousarray(c, dtype=np.int64) for c in coords]
        sec = C.c_double()
        self._check(ref_lib().ref_time_parallel_i64(self._h, _ptrs(cols), cols[0].shape[0], workers,
                                                    C.byref(sec)))
        return sec.value

    def eval_limbs(self, coords, limbs, threads=1):
        """Exact BigInt results as `limbs` uint64 arrays (two's complement)."""
        cols = [np.ascontiguousarray(c, dtype=np.int64) for c in coords]
        n = cols[0].shape[0]
        out = np.zeros((limbs, n), dtype=np.uint64)
        self._check(ref_lib().ref_eval_limbs(self._h, _ptrs(cols), n, limbs, out.ctypes.data,
                                             threads))
        return list(out)

    def eval_interval(self, lo, hi, threads=1):
        lo = [np.ascontiguousarray(c, dtype=np.float64) for c in lo]
        hi = [np.ascontiguousarray(c, dtype=np.float64) for c in hi]
        n = lo[0].shape[0]
        olo, ohi = np.empty(n), np.empty(n)
        self._check(ref_lib().ref_eval_interval(self._h, _ptrs(lo), _ptrs(hi), n, olo.ctypes.data,
                                                ohi.ctypes.data, threads))
        return olo, ohi

    def eval_i64(self, coords, threads=1):
        cols = [np.ascontiguousarray(c, dtype=np.int64) for c in coords]
        out = np.empty(cols[0].shape[0], dtype=np.int64)
        self._check(ref_lib().ref_eval_i64(self._h, _ptrs(cols), out.shape[0], out.ctypes.data,
                                           threads))
        return out

    def dot(self):
        n = C.c_size_t()
        ref_lib().ref_dot(self._h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        ref_lib().ref_dot(self._h, buf, n.value + 1, C.byref(n))
        return buf.value.decode()

    def records(self):
        n, rc = C.c_size_t(), C.c_uint32()
        ref_lib().ref_records(self._h, None, 0, C.byref(n), C.byref(rc))
        buf = np.zeros(5 * max(1, n.value), dtype=np.int32)
        ref_lib().ref_records(self._h, buf.ctypes.data_as(C.POINTER(C.c_int32)), buf.size,
                              C.byref(n), C.byref(rc))
        return buf[: 5 * n.value].reshape(-1, 5), rc.value

    def exponent_set(self, v):
        n = C.c_size_t()
        ref_lib().ref_exponents(self._h, v, None, 0, C.byref(n))
        buf = (C.c_uint32 * max(1, n.value))()
        ref_lib().ref_exponents(self._h, v, buf, n.value, C.byref(n))
        return list(buf)[: n.value]


class ReferenceWide:
    """The unmodified reference BigIntDomain walk with arbitrary-precision
    coefficients and points (the paper's Figure-1 workload), for checking and
    timing pe_eval_wide. Values are little-endian two's-complement words."""

    def __init__(self, exponents, coeff_words, schemes):
        lib = ref_lib()
        e = np.ascontiguousarray(np.asarray(exponents, dtype=np.uint32))
        if e.ndim == 1:
            e = e.reshape(-1, 1)
        w = np.ascontiguousarray(np.asarray(coeff_words, dtype=np.uint64))
        self.nvars = e.shape[1]
        up, lo, cut = _scheme_arrays(schemes)
        h = C.c_void_p()
        self._keep = (e, w)
        if lib.ref_create_wide(e.ctypes.data_as(C.POINTER(C.c_uint32)), w.ctypes.data, w.shape[1],
                               e.shape[0], self.nvars, up, lo, cut, C.byref(h)):
            raise ValueError(lib.ref_last_error().decode())
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                ref_lib().ref_destroy(self._h)
            except Exception:  # noqa: BLE001
                pass
            self._h = None

    def mismatches(self, coords, got, threads=8):
        """Points whose result words `got` (n, out_limbs) differ from the
        reference BigInt result; coords: one (n, point_limbs) array per variable."""
        cols = [np.ascontiguousarray(c, dtype=np.uint64) for c in coords]
        g = np.ascontiguousarray(got, dtype=np.uint64)
        bad = C.c_size_t()
        if ref_lib().ref_eval_wide_check(self._h, _ptrs(cols), cols[0].shape[1], cols[0].shape[0],
                                         g.ctypes.data, g.shape[1], threads, C.byref(bad)):
            raise ValueError(ref_lib().ref_last_error().decode())
        return bad.value

    def seconds(self, coords, threads=1):
        cols = [np.ascontiguousarray(c, dtype=np.uint64) for c in coords]
        t = C.c_double()
        if ref_lib().ref_time_wide(self._h, _ptrs(cols), cols[0].shape[1], cols[0].shape[0], threads,
                                   C.byref(t)):
            raise ValueError(ref_lib().ref_last_error().decode())
        return t.value
