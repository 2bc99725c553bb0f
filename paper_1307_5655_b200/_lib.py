"""ctypes binding of the C ABI in include/polyeval_b200.h.

The shared library is built in-tree (paper_1307_5655_b200/_lib/
libpolyeval_b200.so, see csrc/Makefile and __graft_entry__.build()). There is
no CPU fallback: importing this module without the library raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libpolyeval_b200.so")

PE_OK, PE_EINVAL, PE_EOVERFLOW, PE_ECUDA, PE_ELOGIC = 0, 1, 2, 3, 4

DOMAIN_F64, DOMAIN_F64_STRICT, DOMAIN_I64, DOMAIN_INTERVAL, DOMAIN_I64F = 0, 1, 2, 3, 4


def DOMAIN_LIMBS(k: int) -> int:
    """Domain code of the K-limb exact integer kernel (PE_DOMAIN_LIMBS)."""
    return 0x100 | int(k)

COEFF_F64, COEFF_I64 = 0, 1


class pe_scheme_desc(C.Structure):
    _fields_ = [("upper", C.c_int32), ("lower", C.c_int32), ("cutoff", C.c_uint64)]


class pe_exec(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("strict_f64", C.c_int32),
        ("stream", C.c_void_p),
        ("synchronize", C.c_int32),
        ("i64_int_pipe", C.c_int32),
        ("i64_bounds", C.POINTER(C.c_uint64)),
        ("deferred_checks", C.c_int32),
        ("reserved", C.c_int32),
        ("devices", C.POINTER(C.c_int32)),
        ("ndevices", C.c_int32),
        ("stage_slots", C.c_int32),
        ("stage_chunk", C.c_uint64),
    ]


class pe_tuning(C.Structure):
    """Code-generation options (include/polyeval_b200.h pe_tuning); 0 = default."""
    _fields_ = [
        ("lanes", C.c_uint32),
        ("block", C.c_uint32),
        ("min_ctas", C.c_uint32),
        ("sync_every", C.c_uint32),
        ("section_ops", C.c_uint32),
        ("sched_window", C.c_uint32),
        ("sched_distance", C.c_uint32),
        ("chain_min", C.c_uint32),
        ("iv_fast", C.c_int32),
        ("iv_mid", C.c_int32),
        ("iv_partition", C.c_int32),
        ("group_tiles", C.c_uint32),
        ("word_layout", C.c_int32),
        ("jit_mode", C.c_int32),
        ("iv_partition_min", C.c_uint64),
    ]


class pe_record(C.Structure):
    _fields_ = [
        ("coeff_f64", C.c_double),
        ("coeff_i64", C.c_int64),
        ("sub", C.c_int32),
        ("power_slot", C.c_int32),
        ("lazy_slot", C.c_uint32),
        ("parent_slot", C.c_int32),
        ("reads_register", C.c_int32),
        ("reserved", C.c_int32),
    ]


class pe_compiled_program(C.Structure):
    _fields_ = [
        ("records", C.POINTER(pe_record)),
        ("nrecords", C.c_size_t),
        ("register_count", C.c_uint32),
        ("variable", C.c_uint32),
        ("root_child_ends", C.POINTER(C.c_uint32)),
        ("nroot_child_ends", C.c_size_t),
    ]


class pe_program_info_t(C.Structure):
    _fields_ = [
        ("nvars", C.c_uint32),
        ("register_count", C.c_uint32),
        ("max_registers", C.c_uint32),
        ("records", C.c_uint64),
        ("programs", C.c_uint64),
        ("walk_adds", C.c_uint64),
        ("walk_muls", C.c_uint64),
        ("power_muls", C.c_uint64),
        ("terms", C.c_uint64),
        ("root_children", C.c_uint32),
        ("exponent_set_sizes", C.c_uint32 * 8),
    ]


# (name, restype, argtypes) — must match include/polyeval_b200.h exactly.
EXPORTS = [
    ("pe_program_create", C.c_int,
     [C.POINTER(C.c_uint32), C.c_void_p, C.c_size_t, C.c_uint32,
      C.POINTER(pe_scheme_desc), C.c_int, C.POINTER(C.c_void_p)]),
    ("pe_program_from_compiled", C.c_int,
     [C.POINTER(pe_compiled_program), C.c_size_t, C.c_uint32,
      C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_size_t), C.c_int,
      C.POINTER(C.c_void_p)]),
    ("pe_program_destroy", None, [C.c_void_p]),
    ("pe_program_set_tuning", C.c_int, [C.c_void_p, C.POINTER(pe_tuning)]),
    ("pe_program_info", C.c_int, [C.c_void_p, C.POINTER(pe_program_info_t)]),
    ("pe_program_exponents", C.c_int,
     [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32), C.c_size_t, C.POINTER(C.c_size_t)]),
    ("pe_program_records", C.c_int,
     [C.c_void_p, C.POINTER(C.c_int32), C.c_size_t, C.POINTER(C.c_size_t)]),
    ("pe_program_dot", C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("pe_program_check_registers", C.c_int, [C.c_void_p]),
    ("pe_program_kernel_stats", C.c_int,
     [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
      C.POINTER(C.c_uint64)]),
    ("pe_program_ptx", C.c_int,
     [C.c_void_p, C.c_int32, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("pe_program_compile_only", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64)]),
    ("pe_program_i64_bounds", C.c_int,
     [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("pe_program_f64_slices", C.c_int, [C.c_void_p, C.POINTER(C.c_uint32)]),
    ("pe_program_kernel_ready", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]),
    ("pe_eval_f64", C.c_int,
     [C.c_void_p, C.POINTER(C.c_void_p), C.c_size_t, C.c_void_p, C.POINTER(pe_exec)]),
    ("pe_eval_f64_multi", C.c_int,
     [C.POINTER(C.c_void_p), C.c_size_t, C.POINTER(C.c_void_p), C.c_size_t,
      C.POINTER(C.c_void_p), C.POINTER(pe_exec)]),
    ("pe_eval_i64", C.c_int,
     [C.c_void_p, C.POINTER(C.c_void_p), C.c_size_t, C.c_void_p, C.POINTER(pe_exec)]),
    ("pe_eval_limbs", C.c_int,
     [C.c_void_p, C.POINTER(C.c_void_p), C.c_size_t, C.c_uint32, C.POINTER(C.c_void_p),
      C.POINTER(pe_exec)]),
    ("pe_program_limbs_needed", C.c_int,
     [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]),
    ("pe_eval_interval", C.c_int,
     [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_size_t, C.c_void_p,
      C.c_void_p, C.POINTER(pe_exec)]),
    ("pe_program_create_wide", C.c_int,
     [C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.c_uint32, C.c_size_t, C.c_uint32,
      C.POINTER(pe_scheme_desc), C.POINTER(C.c_void_p)]),
    ("pe_program_wide_limbs", C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32)]),
    ("pe_eval_wide", C.c_int,
     [C.c_void_p, C.POINTER(C.c_void_p), C.c_uint32, C.c_size_t, C.c_void_p, C.c_uint32,
      C.POINTER(pe_exec)]),
    ("pe_measure_peak", C.c_int,
     [C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
    ("pe_synchronize", C.c_int, [C.POINTER(pe_exec)]),
    ("pe_launch_count", C.c_uint64, []),
    ("pe_last_error", C.c_char_p, []),
    ("pe_version", C.c_char_p, []),
]

_lib = None


def lib():
    """Loads the library once; raises ImportError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"polyeval-b200 native library missing at {LIB_PATH}; "
            "run `python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
    handle = C.CDLL(LIB_PATH)
    for name, res, args in EXPORTS:
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _lib = handle
    return _lib


class PolyEvalError(RuntimeError):
    """Base class; subclasses mirror the reference exception taxonomy."""


class CudaError(PolyEvalError):
    pass


class LogicError(PolyEvalError):
    """std::logic_error analogue (e.g. register hygiene / internal)."""


def check(status: int) -> None:
    if status == PE_OK:
        return
    msg = lib().pe_last_error().decode(errors="replace")
    if status == PE_EINVAL:
        raise ValueError(msg)
    if status == PE_EOVERFLOW:
        raise OverflowError(msg)
    if status == PE_ECUDA:
        raise CudaError(msg)
    raise LogicError(msg)
