"""Host-side mirror of the reference's compile-once / evaluate API.

Reference interface (proj/core/include/polyeval/):
  scheme.hpp:15-57   FunctionScheme, builtin_scheme, threshold_combine
  polynomial.hpp     Polynomial (canonical sparse terms)
  tree.hpp:58-88     build / build_multivariate / compute_lazy_heights / to_dot
  eval.hpp:32-57     CompiledProgram, compile(tree)
  eval.hpp:69-90     Evaluator<D>(domain, program).evaluate(point)
  ring.hpp:30-65     BigIntDomain / DoubleDomain / IntervalDomain

Differences, by design: `evaluate` takes a *batch* of points (structure of
arrays, one array per variable) and runs on the GPU through the C ABI; the
BigInt domain is the exact int64 path with a host overflow proof
(OverflowError instead of wrapping). Errors follow the reference taxonomy:
ValueError <=> std::invalid_argument, LogicError <=> std::logic_error.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib as L


# ----------------------------------------------------------------- schemes

class BuiltinScheme(enum.IntEnum):
    direct = 0
    horner = 1
    estrin = 2
    balanced = 3


@dataclass(frozen=True)
class FunctionScheme:
    """A scheme is `upper` alone (cutoff 0) or threshold_combine(upper, lower, cutoff)."""
    upper: BuiltinScheme
    lower: BuiltinScheme = BuiltinScheme.horner
    cutoff: int = 0

    @property
    def name(self) -> str:
        if self.cutoff == 0:
            return self.upper.name
        return f"{self.upper.name}:{self.lower.name}@{self.cutoff}"

    def split(self, k: int) -> int:
        """Python restatement of the split function (reference scheme.cpp:10-34)."""
        which = self.upper if (self.cutoff == 0 or k > self.cutoff) else self.lower
        if which == BuiltinScheme.direct:
            return k
        if which == BuiltinScheme.horner:
            return 1
        if which == BuiltinScheme.estrin:
            return 1 << (k.bit_length() - 1) if k > 0 else 0
        return (k + 1) // 2

    def desc(self) -> L.pe_scheme_desc:
        return L.pe_scheme_desc(int(self.upper), int(self.lower), int(self.cutoff))


def builtin_scheme(which) -> FunctionScheme:
    if isinstance(which, str):
        which = BuiltinScheme[which]
    return FunctionScheme(BuiltinScheme(which))


def threshold_combine(upper: FunctionScheme, lower: FunctionScheme, cutoff: int) -> FunctionScheme:
    if cutoff < 1:
        raise ValueError("threshold cutoff must be >= 1")
    if upper.cutoff or lower.cutoff:
        raise ValueError("nested threshold schemes are not expressible across the C ABI")
    return FunctionScheme(upper.upper, lower.upper, int(cutoff))


def scheme_from_name(name: str) -> FunctionScheme:
    """'name' or 'upper:lower@N' (reference tools/scheme_name.cpp:34-53)."""
    if ":" not in name:
        return builtin_scheme(name)
    up, rest = name.split(":", 1)
    if "@" not in rest:
        raise ValueError(f"bad scheme name {name!r}")
    lo, cut = rest.split("@", 1)
    if not cut.isdigit() or int(cut) < 1:
        raise ValueError(f"bad scheme cutoff in {name!r}")
    return threshold_combine(builtin_scheme(up), builtin_scheme(lo), int(cut))


# ----------------------------------------------------------------- polynomial

@dataclass
class Polynomial:
    """Raw terms: exponents (T, V) uint32 and coefficients (T,) float64|int64.

    Canonicalisation (sort, merge like terms, drop zeros) happens in the
    native front-end at compile time (reference polynomial.cpp:13-33).
    """
    exponents: np.ndarray
    coefficients: np.ndarray
    variables: tuple = ("x",)

    def __post_init__(self):
        # range checks before any cast: astype would wrap silently
        e = np.asarray(self.exponents)
        if e.dtype.kind not in "iu":
            if e.dtype.kind == "f" and np.all(np.isfinite(e)) and np.all(e == np.floor(e)):
                e = e.astype(np.float64)
            elif e.dtype != object:
                raise ValueError("exponents must be integers")
        if e.size:
            lo, hi = (int(e.min()), int(e.max())) if e.dtype != object else \
                (min(int(v) for v in e.flat), max(int(v) for v in e.flat))
            if lo < 0 or hi >= 2**32:
                raise ValueError("exponents must lie in [0, 2^32)")
        self.exponents = np.ascontiguousarray(np.asarray(e).astype(np.int64).astype(np.uint32))
        if self.exponents.ndim == 1:
            self.exponents = self.exponents.reshape(-1, 1)
        c = np.asarray(self.coefficients)
        if c.dtype == object and all(isinstance(v, (int, np.integer)) for v in c.flat):
            c = np.asarray([int(v) for v in c.flat], dtype=object).reshape(c.shape)
            if c.size and (min(c.flat) < -2**63 or max(c.flat) >= 2**63):
                raise OverflowError("integer coefficients must fit int64")
            c = c.astype(np.int64)
        elif c.dtype.kind == "u":
            if c.size and int(c.max()) >= 2**63:
                raise OverflowError("integer coefficients must fit int64")
            c = c.astype(np.int64)
        elif c.dtype.kind == "i":
            c = c.astype(np.int64)
        else:
            c = c.astype(np.float64)
        self.coefficients = np.ascontiguousarray(c)
        if self.exponents.shape[0] != self.coefficients.shape[0]:
            raise ValueError("one coefficient per term")
        if len(self.variables) != self.exponents.shape[1]:
            self.variables = tuple("xyz"[i] if self.exponents.shape[1] <= 3 else f"x{i}"
                                   for i in range(self.exponents.shape[1]))

    @property
    def nvars(self) -> int:
        return self.exponents.shape[1]

    @classmethod
    def univariate(cls, coeffs_high_to_low, dtype=None) -> "Polynomial":
        """Dense univariate from coefficients c_d..c_0 (highest degree first)."""
        c = np.asarray(coeffs_high_to_low, dtype=dtype)
        d = len(c) - 1
        return cls(np.arange(d, -1, -1, dtype=np.uint32).reshape(-1, 1), c, ("x",))


# ----------------------------------------------------------------- program

_DEFAULT_TUNING: dict = {}


def set_default_tuning(**options) -> None:
    """pe_tuning fields applied to every program compiled afterwards in this
    process (e.g. jit_mode=1: calls wait for the specialised kernel instead
    of running the walk VM while it compiles). No arguments: defaults."""
    names = {f for f, _ in L.pe_tuning._fields_}
    for k in options:
        if k not in names:
            raise ValueError(f"unknown tuning option {k!r}")
    _DEFAULT_TUNING.clear()
    _DEFAULT_TUNING.update(options)


class CompiledProgram:
    """Owns a native pe_program (immutable, shareable across threads)."""

    def __init__(self, poly: Polynomial, schemes: Sequence[FunctionScheme]):
        lib = L.lib()
        if len(schemes) != poly.nvars:
            raise ValueError("need exactly one scheme per variable")
        self.poly = poly
        self.schemes = tuple(schemes)
        self._nvars = poly.nvars
        self.integer = poly.coefficients.dtype == np.int64
        descs = (L.pe_scheme_desc * poly.nvars)(*[s.desc() for s in schemes])
        h = C.c_void_p()
        st = lib.pe_program_create(
            poly.exponents.ctypes.data_as(C.POINTER(C.c_uint32)),
            poly.coefficients.ctypes.data_as(C.c_void_p), poly.coefficients.shape[0],
            poly.nvars, descs, L.COEFF_I64 if self.integer else L.COEFF_F64, C.byref(h))
        L.check(st)
        self._h = h
        if _DEFAULT_TUNING:
            self.set_tuning(**_DEFAULT_TUNING)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                L.lib().pe_program_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def nvars(self) -> int:
        return self._nvars

    @classmethod
    def from_compiled(cls, programs, exponent_sets, integer: bool = False) -> "CompiledProgram":
        """Lowers an already compiled program (pe_program_from_compiled).

        programs: list of dicts, [0] the root, each {"records": [dict(coeff,
        sub, power_slot, lazy_slot, parent_slot, reads_register)],
        "register_count", "variable", "root_child_ends"}; `sub` / `power_slot`
        / `parent_slot` are -1 when absent (reference CompiledProgram,
        eval.hpp:32-54). exponent_sets: one ascending list per variable."""
        nvars = len(exponent_sets)
        keep = []
        progs = (L.pe_compiled_program * len(programs))()
        for k, pr in enumerate(programs):
            recs = (L.pe_record * len(pr["records"]))()
            for i, r in enumerate(pr["records"]):
                if integer:
                    recs[i].coeff_i64 = int(r.get("coeff", 0))
                else:
                    recs[i].coeff_f64 = float(r.get("coeff", 0.0))
                recs[i].sub = int(r.get("sub", -1))
                recs[i].power_slot = int(r.get("power_slot", -1))
                recs[i].lazy_slot = int(r["lazy_slot"])
                recs[i].parent_slot = int(r.get("parent_slot", -1))
                recs[i].reads_register = 1 if r.get("reads_register") else 0
            ends = (C.c_uint32 * max(1, len(pr.get("root_child_ends", []))))(
                *pr.get("root_child_ends", []))
            keep += [recs, ends]
            progs[k].records = recs
            progs[k].nrecords = len(pr["records"])
            progs[k].register_count = int(pr["register_count"])
            progs[k].variable = int(pr.get("variable", 0))
            progs[k].root_child_ends = ends
            progs[k].nroot_child_ends = len(pr.get("root_child_ends", []))
        sets = [(C.c_uint32 * max(1, len(e)))(*e) for e in exponent_sets]
        set_ptrs = (C.POINTER(C.c_uint32) * nvars)(*[C.cast(a, C.POINTER(C.c_uint32)) for a in sets])
        sizes = (C.c_size_t * nvars)(*[len(e) for e in exponent_sets])
        h = C.c_void_p()
        L.check(L.lib().pe_program_from_compiled(progs, len(programs), nvars, set_ptrs, sizes,
                                                 L.COEFF_I64 if integer else L.COEFF_F64,
                                                 C.byref(h)))
        self = cls.__new__(cls)
        self.poly = None
        self.schemes = ()
        self._nvars = nvars
        self.integer = bool(integer)
        self._h = h
        if _DEFAULT_TUNING:
            self.set_tuning(**_DEFAULT_TUNING)
        return self

    def limbs_needed(self, bounds) -> int:
        """Smallest K (1..8) of 64-bit limbs the overflow proof allows for
        |x_v| <= bounds[v]; 0 if more than 8 would be needed."""
        b = (C.c_uint64 * self.nvars)(*[int(x) for x in bounds])
        k = C.c_uint32()
        L.check(L.lib().pe_program_limbs_needed(self._h, b, C.byref(k)))
        return k.value

    def info(self) -> dict:
        inf = L.pe_program_info_t()
        L.check(L.lib().pe_program_info(self._h, C.byref(inf)))
        return {
            "nvars": inf.nvars, "register_count": inf.register_count,
            "max_registers": inf.max_registers, "records": inf.records,
            "programs": inf.programs, "walk_adds": inf.walk_adds, "walk_muls": inf.walk_muls,
            "power_muls": inf.power_muls, "terms": inf.terms,
            "root_children": inf.root_children,
            "exponent_set_sizes": list(inf.exponent_set_sizes)[: inf.nvars],
        }

    def exponent_set(self, v: int) -> list:
        n = C.c_size_t()
        L.check(L.lib().pe_program_exponents(self._h, v, None, 0, C.byref(n)))
        buf = (C.c_uint32 * max(1, n.value))()
        L.check(L.lib().pe_program_exponents(self._h, v, buf, n.value, C.byref(n)))
        return list(buf)[: n.value]

    def records(self) -> np.ndarray:
        """(records, 5): power_slot|-1, lazy_slot, parent_slot|-1, reads_register, has_sub."""
        n = C.c_size_t()
        L.check(L.lib().pe_program_records(self._h, None, 0, C.byref(n)))
        buf = np.zeros(5 * max(1, n.value), dtype=np.int32)
        L.check(L.lib().pe_program_records(
            self._h, buf.ctypes.data_as(C.POINTER(C.c_int32)), buf.size, C.byref(n)))
        return buf[: 5 * n.value].reshape(-1, 5)

    def dot(self) -> str:
        n = C.c_size_t()
        L.check(L.lib().pe_program_dot(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        L.check(L.lib().pe_program_dot(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def ptx(self, domain: int) -> str:
        n = C.c_size_t()
        L.check(L.lib().pe_program_ptx(self._h, domain, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        L.check(L.lib().pe_program_ptx(self._h, domain, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def kernel_stats(self, domain: int) -> dict:
        fp, it, nb = C.c_uint64(), C.c_uint64(), C.c_uint64()
        L.check(L.lib().pe_program_kernel_stats(self._h, domain, C.byref(fp), C.byref(it),
                                                C.byref(nb)))
        return {"fp_ops": fp.value, "int_ops": it.value, "ptx_bytes": nb.value}

    def i64_bounds(self):
        """(bound63, bound53): per-variable coordinate bounds for the exact
        int64 kernel and the faster exact-on-FP64 tier."""
        b63 = (C.c_uint64 * self.nvars)()
        b53 = (C.c_uint64 * self.nvars)()
        L.check(L.lib().pe_program_i64_bounds(self._h, b63, b53))
        return list(b63), list(b53)

    def f64_slices(self) -> int:
        k = C.c_uint32()
        L.check(L.lib().pe_program_f64_slices(self._h, C.byref(k)))
        return k.value

    def set_tuning(self, **options) -> None:
        """Code-generation options (pe_tuning fields, e.g. lanes=2,
        section_ops=4000, iv_fast=-1, jit_mode=1); drops the generated
        kernels. Fields not given are the process defaults
        (set_default_tuning), then the library's."""
        options = {**_DEFAULT_TUNING, **options}
        t = L.pe_tuning()
        names = {f for f, _ in L.pe_tuning._fields_}
        for k, v in options.items():
            if k not in names:
                raise ValueError(f"unknown tuning option {k!r}")
            setattr(t, k, int(v))
        L.check(L.lib().pe_program_set_tuning(self._h, C.byref(t)))

    def kernel_ready(self, domain: int) -> bool:
        """True once the specialised kernel of `domain` is compiled (until
        then calls run the walk VM, pe_tuning.jit_mode 0)."""
        r = C.c_int32()
        L.check(L.lib().pe_program_kernel_ready(self._h, domain, C.byref(r)))
        return bool(r.value)

    def compile_only(self, domain: int) -> int:
        nb = C.c_uint64()
        L.check(L.lib().pe_program_compile_only(self._h, domain, C.byref(nb)))
        return nb.value


def compile(poly: Polynomial, schemes) -> CompiledProgram:  # noqa: A001 (reference name)
    """build/build_multivariate + compute_lazy_heights + compile in one call."""
    if isinstance(schemes, FunctionScheme):
        schemes = [schemes] * poly.nvars
    return CompiledProgram(poly, schemes)


# ----------------------------------------------------------------- domains

class DoubleDomain:
    """fp64; strict=True replays the reference op order bit-exactly."""
    def __init__(self, strict: bool = False):
        self.strict = bool(strict)


class IntervalDomain:
    """Reference IntervalDomain: RN op + one nextafter step outward."""


class BigIntDomain:
    """Exact integer domain on a host-proven range.

    By default the runtime evaluates on the FP64 FMA pipe whenever the host
    proves every intermediate stays below 2^53 (exact), else with int64
    multiply-adds; int_pipe=True forces the int64 kernel. wide=True lifts the
    int64 limit: values are carried in K 64-bit limbs (K = the smallest the
    proof allows for the batch, up to 8 = 511-bit values) and evaluate()
    returns Python ints (pe_eval_limbs)."""

    def __init__(self, int_pipe: bool = False, wide: bool = False):
        self.int_pipe = bool(int_pipe)
        self.wide = bool(wide)


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _check_tensor(t, dtype, what):
    """A CUDA tensor is handed to the kernels as a raw pointer: its element
    type must be exactly the domain's (float32 data read as float64 would run
    past the buffer)."""
    import torch
    want = torch.float64 if np.dtype(dtype) == np.float64 else torch.int64
    if t.dtype != want:
        raise TypeError(f"{what} tensor must have dtype {want}, got {t.dtype}")
    if t.dim() != 1:
        raise ValueError(f"{what} tensor must be one-dimensional")


class Evaluator:
    """Batch evaluation session (reference Evaluator<D>, eval.hpp:69-90)."""

    def __init__(self, domain, program: CompiledProgram, device: int = -1,
                 deferred_checks: bool = False, synchronize: bool = False,
                 devices: Sequence[int] | None = None):
        """CUDA-tensor calls are asynchronous on the stream they are enqueued
        on (torch's current stream of the data's device unless `stream=` is
        given), like any torch CUDA op; `synchronize=True` waits for the
        result before returning. Host (numpy) calls always return finished
        results.

        deferred_checks: device-pointer int64 / interval calls return
        without a host round trip; domain-check failures surface at
        `synchronize()` (pe_exec.deferred_checks).

        devices: host (numpy) batches are split into contiguous slices, one
        per listed GPU, evaluated concurrently and written straight into the
        host result (pe_exec.devices)."""
        self.domain = domain
        self.program = program
        self.device = device
        self.deferred_checks = bool(deferred_checks)
        self.sync = bool(synchronize)
        self.devices = [int(d) for d in devices] if devices else []
        self._dev_arr = (C.c_int32 * max(1, len(self.devices)))(*self.devices)
        if isinstance(domain, BigIntDomain) and not program.integer:
            raise ValueError("BigIntDomain needs integer coefficients")

    def _exec(self, stream=None, sync=None, bounds=None) -> L.pe_exec:
        ex = L.pe_exec()
        ex.device = self.device
        ex.strict_f64 = 1 if isinstance(self.domain, DoubleDomain) and self.domain.strict else 0
        ex.stream = stream
        ex.synchronize = 1 if (self.sync if sync is None else sync) else 0
        ex.i64_int_pipe = 1 if isinstance(self.domain, BigIntDomain) and self.domain.int_pipe else 0
        ex.deferred_checks = 1 if self.deferred_checks else 0
        if self.devices:
            ex.devices = C.cast(self._dev_arr, C.POINTER(C.c_int32))
            ex.ndevices = len(self.devices)
        if bounds is not None:
            arr = (C.c_uint64 * len(bounds))(*[int(b) for b in bounds])
            ex.i64_bounds = arr
            self._keep = arr
        return ex

    def _soa(self, points, dtype):
        if isinstance(points, np.ndarray) and points.ndim == 2:
            if points.shape[1] != self.program.nvars:
                raise ValueError("evaluation point arity mismatch")
            points = [points[:, v] for v in range(points.shape[1])]
        if len(points) != self.program.nvars:
            raise ValueError("evaluation point arity mismatch")
        cols = []
        on_gpu = [_is_torch_cuda(p) for p in points]
        if any(on_gpu) and not all(on_gpu):
            raise ValueError("coordinates must be all CUDA tensors or all host arrays")
        for p in points:
            if _is_torch_cuda(p):
                _check_tensor(p, dtype, "coordinate")
                if p.device != points[0].device:
                    raise ValueError("all coordinate tensors must be on one device")
                if not p.is_contiguous():
                    p = p.contiguous()
                cols.append(p)
            else:
                cols.append(np.ascontiguousarray(np.asarray(p, dtype=dtype)))
        n = {int(c.shape[0]) for c in cols}
        if len(n) != 1:
            raise ValueError("all coordinate arrays must have the same length")
        return cols, n.pop()

    @staticmethod
    def _check_out(out, dtype, n, like):
        """out= must live where the coordinates do, with the result dtype."""
        if _is_torch_cuda(like):
            if not _is_torch_cuda(out):
                raise ValueError("out must be a CUDA tensor for CUDA coordinates")
            _check_tensor(out, dtype, "out")
            if out.device != like.device:
                raise ValueError("out must be on the coordinates' device")
            if not out.is_contiguous():
                raise ValueError("out must be contiguous")
        else:
            if not isinstance(out, np.ndarray):
                raise ValueError("out must be a numpy array for host coordinates")
            if out.dtype != np.dtype(dtype):
                raise TypeError(f"out must have dtype {np.dtype(dtype)}, got {out.dtype}")
            if not out.flags.c_contiguous or not out.flags.writeable:
                raise ValueError("out must be a writeable contiguous array")
        if int(out.shape[0]) != n or len(out.shape) != 1:
            raise ValueError(f"out must have shape ({n},)")

    @staticmethod
    def _ptr(a):
        return a.data_ptr() if _is_torch_cuda(a) else a.ctypes.data

    def evaluate(self, points, out=None, stream=None, bounds=None):
        """points: per-variable arrays (numpy -> host staged, torch CUDA ->
        in place); IntervalDomain takes (lo_arrays, hi_arrays)."""
        lib = L.lib()
        self._register_check()
        if isinstance(self.domain, IntervalDomain):
            lo, hi = points
            lo_c, n = self._soa(lo, np.float64)
            hi_c, n2 = self._soa(hi, np.float64)
            if n != n2:
                raise ValueError("lo/hi length mismatch")
            dev = _is_torch_cuda(lo_c[0])
            if dev != _is_torch_cuda(hi_c[0]) or (dev and hi_c[0].device != lo_c[0].device):
                raise ValueError("lo and hi must live on the same device")
            if out is None:
                out = (self._alloc(n, "f64", dev, lo_c[0]), self._alloc(n, "f64", dev, lo_c[0]))
            for o in out:
                self._check_out(o, np.float64, n, lo_c[0])
            lo_p = (C.c_void_p * len(lo_c))(*[self._ptr(a) for a in lo_c])
            hi_p = (C.c_void_p * len(hi_c))(*[self._ptr(a) for a in hi_c])
            ex = self._exec(self._stream(stream, lo_c[0]))
            L.check(lib.pe_eval_interval(self.program.handle, lo_p, hi_p, n, self._ptr(out[0]),
                                         self._ptr(out[1]), C.byref(ex)))
            return out
        integer = isinstance(self.domain, BigIntDomain)
        if integer and self.domain.wide:
            k, limbs = self.evaluate_limbs(points, stream=stream)
            return limbs_to_int(limbs)
        cols, n = self._soa(points, np.int64 if integer else np.float64)
        dev = _is_torch_cuda(cols[0])
        if out is None:
            out = self._alloc(n, "i64" if integer else "f64", dev, cols[0])
        self._check_out(out, np.int64 if integer else np.float64, n, cols[0])
        ptrs = (C.c_void_p * len(cols))(*[self._ptr(a) for a in cols])
        ex = self._exec(self._stream(stream, cols[0]), bounds=bounds)
        fn = lib.pe_eval_i64 if integer else lib.pe_eval_f64
        L.check(fn(self.program.handle, ptrs, n, self._ptr(out), C.byref(ex)))
        return out

    def evaluate_limbs(self, points, limbs: int | None = None, stream=None):
        """K-limb exact evaluation (pe_eval_limbs): returns (K, [K arrays of
        uint64 words, little-endian two's complement]); K defaults to the
        smallest the overflow proof allows for this batch's coordinates."""
        cols, n = self._soa(points, np.int64)
        dev = _is_torch_cuda(cols[0])
        if limbs is None:
            maxima = []
            for c in cols:
                if dev:
                    maxima.append(int(c.abs().max().item()) if n else 0)
                else:
                    maxima.append(int(np.abs(c.astype(np.int64)).max()) if n else 0)
            maxima = [min(m, 2**63) for m in maxima]
            limbs = self.program.limbs_needed(maxima)
            if limbs == 0:
                raise OverflowError("values need more than 8 limbs (511 bits)")
        outs = [Evaluator._alloc(n, "i64", dev, cols[0]) for _ in range(limbs)]
        ptrs = (C.c_void_p * len(cols))(*[self._ptr(a) for a in cols])
        optrs = (C.c_void_p * limbs)(*[self._ptr(o) for o in outs])
        ex = self._exec(self._stream(stream, cols[0]))
        L.check(L.lib().pe_eval_limbs(self.program.handle, ptrs, n, limbs, optrs, C.byref(ex)))
        if not dev:
            outs = [o.view(np.uint64) for o in outs]
        return limbs, outs

    def enable_register_check(self, on: bool = True) -> None:
        """Reference Evaluator::enable_register_check (eval.hpp:142-145):
        evaluate() raises LogicError if the walk leaves a value unconsumed.
        Every point walks the same records, so the check runs once per
        program, symbolically (pe_program_check_registers)."""
        self.check_registers = bool(on)
        self._registers_ok = None

    def _register_check(self):
        if getattr(self, "check_registers", False):
            if self._registers_ok is None:
                L.check(L.lib().pe_program_check_registers(self.program.handle))
                self._registers_ok = True

    def evaluate_parallel(self, points, workers: int, out=None, stream=None):
        """Reference evaluate_parallel (eval.hpp:97-140): same result as
        evaluate() — bit-identical by the reference's own contract — with the
        worker count validated; the batch is already spread over the GPU."""
        if int(workers) < 1:
            raise ValueError("workers must be >= 1")
        return self.evaluate(points, out=out, stream=stream)

    def synchronize(self, stream=None):
        """Waits for the stream; raises any deferred domain-check failure."""
        import torch
        if stream is None:
            dev = torch.device("cuda", self.device) if self.device >= 0 else None
            stream = torch.cuda.current_stream(dev).cuda_stream
        ex = self._exec(stream)
        L.check(L.lib().pe_synchronize(C.byref(ex)))

    @staticmethod
    def _stream(stream, like):
        """Explicit stream, else torch's current stream on the data's device."""
        if stream is not None:
            return stream
        if like is not None and _is_torch_cuda(like):
            import torch
            return torch.cuda.current_stream(like.device).cuda_stream
        return None

    @staticmethod
    def _alloc(n, kind, dev, like):
        if dev:
            import torch
            dt = torch.int64 if kind == "i64" else torch.float64
            return torch.empty(n, dtype=dt, device=like.device)
        return np.empty(n, dtype=np.int64 if kind == "i64" else np.float64)


def evaluate_many(programs, points, outs=None, device: int = -1, stream=None, devices=None):
    """Fused-fp64 evaluation of several programs over one batch
    (pe_eval_f64_multi): host points are staged to the GPU once."""
    ev = Evaluator(DoubleDomain(), programs[0], device=device, devices=devices)
    cols, n = ev._soa(points, np.float64)
    dev = _is_torch_cuda(cols[0])
    if outs is None:
        outs = [Evaluator._alloc(n, "f64", dev, cols[0]) for _ in programs]
    if len(outs) != len(programs):
        raise ValueError("one output per program")
    for o in outs:
        Evaluator._check_out(o, np.float64, n, cols[0])
    handles = (C.c_void_p * len(programs))(*[p.handle.value for p in programs])
    ptrs = (C.c_void_p * len(cols))(*[Evaluator._ptr(a) for a in cols])
    optrs = (C.c_void_p * len(outs))(*[Evaluator._ptr(o) for o in outs])
    ex = ev._exec(Evaluator._stream(stream, cols[0]))
    L.check(L.lib().pe_eval_f64_multi(handles, len(programs), ptrs, n, optrs, C.byref(ex)))
    return outs


def evaluate(program: CompiledProgram, points, domain):
    """One-shot convenience wrapper (reference eval.hpp:262-268)."""
    return Evaluator(domain, program).evaluate(points)


def limbs_to_int(limbs) -> np.ndarray:
    """K arrays of 64-bit words (little-endian two's complement) -> object
    array of Python ints."""
    host = [np.asarray(l.cpu() if hasattr(l, "cpu") else l).view(np.uint64) for l in limbs]
    k = len(host)
    out = np.empty(host[0].shape[0], dtype=object)
    top = 1 << (64 * k)
    for i in range(out.shape[0]):
        v = 0
        for j in range(k - 1, -1, -1):
            v = (v << 64) | int(host[j][i])
        out[i] = v - top if v >> (64 * k - 1) else v
    return out


def evaluate_parallel(program: CompiledProgram, points, domain, workers: int):
    """One-shot parallel evaluation (reference eval.hpp:271-277)."""
    return Evaluator(domain, program).evaluate_parallel(points, workers)


# ----------------------------------------------------------------- wide integers

def ints_to_words(values, limbs: int) -> np.ndarray:
    """Python ints -> (n, limbs) uint64 words, little-endian two's complement.
    Raises OverflowError if a value needs more than 64 * limbs - 1 bits."""
    vals = [int(v) for v in values]
    out = np.zeros((len(vals), limbs), dtype=np.uint64)
    top = 1 << (64 * limbs)
    for i, v in enumerate(vals):
        if not -(top >> 1) <= v < (top >> 1):
            raise OverflowError(f"value needs more than {64 * limbs - 1} bits")
        u = v % top
        for k in range(limbs):
            out[i, k] = (u >> (64 * k)) & 0xFFFFFFFFFFFFFFFF
    return out


def words_to_ints(words) -> list:
    """(n, limbs) uint64 two's-complement words -> Python ints."""
    w = np.asarray(words, dtype=np.uint64)
    limbs = w.shape[1]
    top = 1 << (64 * limbs)
    out = []
    for row in w:
        v = 0
        for k in range(limbs - 1, -1, -1):
            v = (v << 64) | int(row[k])
        out.append(v - top if v >> (64 * limbs - 1) else v)
    return out


def limbs_for(values) -> int:
    """Smallest limb count holding every value in two's complement."""
    bits = max((abs(int(v)).bit_length() for v in values), default=0)
    return max(1, (bits + 1 + 63) // 64)


def compile_wide(exponents, coefficients, schemes) -> CompiledProgram:
    """A program with arbitrary-precision integer coefficients (Python ints;
    the reference's BigInt Polynomial), evaluated by evaluate_wide — the
    paper's Figure-1 workload (pe_program_create_wide). Exponent rows must be
    distinct."""
    e = np.ascontiguousarray(np.asarray(exponents, dtype=np.int64))
    if e.ndim == 1:
        e = e.reshape(-1, 1)
    if e.size and (e.min() < 0 or e.max() >= 2**32):
        raise ValueError("exponents must lie in [0, 2^32)")
    e = np.ascontiguousarray(e.astype(np.uint32))
    nvars = e.shape[1]
    if isinstance(schemes, FunctionScheme):
        schemes = [schemes] * nvars
    if len(schemes) != nvars:
        raise ValueError("need exactly one scheme per variable")
    coefs = [int(c) for c in coefficients]
    if len(coefs) != e.shape[0]:
        raise ValueError("one coefficient per term")
    limbs = limbs_for(coefs)
    words = np.ascontiguousarray(ints_to_words(coefs, limbs))
    descs = (L.pe_scheme_desc * nvars)(*[s.desc() for s in schemes])
    h = C.c_void_p()
    L.check(L.lib().pe_program_create_wide(e.ctypes.data_as(C.POINTER(C.c_uint32)),
                                           words.ctypes.data_as(C.POINTER(C.c_uint64)), limbs,
                                           e.shape[0], nvars, descs, C.byref(h)))
    self = CompiledProgram.__new__(CompiledProgram)
    self.poly = None
    self.schemes = tuple(schemes)
    self._nvars = nvars
    self.integer = True
    self._h = h
    self.wide = True
    return self


def wide_limbs(program: CompiledProgram, point_limbs: int) -> int:
    """Result limbs the static bound needs for points of point_limbs words."""
    k = C.c_uint32()
    L.check(L.lib().pe_program_wide_limbs(program.handle, point_limbs, C.byref(k)))
    return k.value


def evaluate_wide(program: CompiledProgram, points, point_limbs: int | None = None,
                  device: int = -1, as_words: bool = False):
    """Exact evaluation at integer points of any size (pe_eval_wide, one warp
    per point on large batches). points: one sequence of Python ints per variable, or one
    (n, point_limbs) uint64 word array per variable. Returns Python ints (or
    the (n, out_limbs) result words with as_words=True)."""
    if len(points) != program.nvars:
        raise ValueError("evaluation point arity mismatch")
    cols = []
    if point_limbs is None:
        if all(isinstance(p, np.ndarray) and p.ndim == 2 for p in points):
            point_limbs = points[0].shape[1]
        else:
            point_limbs = max(limbs_for(p) for p in points)
    for p in points:
        if isinstance(p, np.ndarray) and p.ndim == 2:
            if p.shape[1] != point_limbs or p.dtype != np.uint64:
                raise ValueError("word arrays must be (n, point_limbs) uint64")
            cols.append(np.ascontiguousarray(p))
        else:
            cols.append(np.ascontiguousarray(ints_to_words(p, point_limbs)))
    n = {c.shape[0] for c in cols}
    if len(n) != 1:
        raise ValueError("all coordinate arrays must have the same length")
    n = n.pop()
    out_limbs = wide_limbs(program, point_limbs)
    out = np.zeros((n, out_limbs), dtype=np.uint64)
    ptrs = (C.c_void_p * len(cols))(*[c.ctypes.data for c in cols])
    ex = L.pe_exec()
    ex.device = device
    L.check(L.lib().pe_eval_wide(program.handle, ptrs, point_limbs, n, out.ctypes.data, out_limbs,
                                 C.byref(ex)))
    return out if as_words else words_to_ints(out)


def launch_count() -> int:
    return int(L.lib().pe_launch_count())
