"""pe_program_from_compiled: lowering an existing reference CompiledProgram.

The reference's own compile() output (exported by oracle/ref_harness.cpp from
the unmodified library) goes through pe_program_from_compiled; the generated
kernels must be identical to the ones pe_program_create builds from the raw
terms (our front-end reproduces the reference compile()), and malformed
programs must be rejected (pe_program_from_compiled).
"""
import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W
import pyoracle

needs_ref = pytest.mark.skipif(not pyoracle.ref_available(), reason="oracle/_ref not built")

CASES = {
    "c1": W.c1, "c2e1000": lambda: W.c2(1000, "estrin"), "c2b1023": lambda: W.c2(1023, "balanced"),
    "c3": W.c3, "c5": W.c5,
}


def _domains(wl):
    if wl.domain == "i64":
        return [pe.DOMAIN_I64, pe.DOMAIN_I64F]
    return [pe.DOMAIN_F64, pe.DOMAIN_F64_STRICT, pe.DOMAIN_INTERVAL]


@needs_ref
@pytest.mark.parametrize("name", list(CASES))
def test_reference_compiled_program_lowers_to_identical_kernels(name):
    wl = CASES[name]()
    progs, sets = pyoracle.Reference(wl.poly, wl.schemes).export()
    imported = pe.CompiledProgram.from_compiled(progs, sets, integer=wl.domain == "i64")
    native = pe.compile(wl.poly, wl.schemes)
    assert imported.info() == native.info()
    for d in _domains(wl):
        assert imported.ptx(d) == native.ptx(d)
    if wl.domain == "i64":
        assert imported.i64_bounds() == native.i64_bounds()


@needs_ref
def test_reference_compiled_trivariate_nested_programs():
    wl = W.c4()
    progs, sets = pyoracle.Reference(wl.poly, wl.schemes).export()
    assert len(progs) > 2000  # root + nested y- and z-programs
    imported = pe.CompiledProgram.from_compiled(progs, sets)
    native = pe.compile(wl.poly, wl.schemes)
    assert imported.info() == native.info()
    assert imported.ptx(pe.DOMAIN_F64) == native.ptx(pe.DOMAIN_F64)
    # sections are cut on the lowered op stream, so the reference's own
    # CompiledProgram gets the identical sectioned kernel
    assert imported.f64_slices() == native.f64_slices() > 1
    with pytest.raises(ValueError):
        imported.dot()


def _horner_3x2_2x_1():
    # 3x^2 + 2x + 1 by Hörner, written by hand in the reference layout
    return ([{"records": [
        {"coeff": 3.0, "power_slot": 0, "lazy_slot": 0, "parent_slot": 0},
        {"coeff": 2.0, "power_slot": 0, "lazy_slot": 0, "parent_slot": 0, "reads_register": True},
        {"coeff": 1.0, "lazy_slot": 0, "reads_register": True},
    ], "register_count": 1, "variable": 0, "root_child_ends": [1]}], [[1]])


def test_hand_written_program_compiles():
    progs, sets = _horner_3x2_2x_1()
    prog = pe.CompiledProgram.from_compiled(progs, sets)
    inf = prog.info()
    assert inf["records"] == 3 and inf["walk_muls"] == 2
    assert prog.compile_only(pe.DOMAIN_F64) > 0
    assert prog.compile_only(pe.DOMAIN_INTERVAL) > 0


@pytest.mark.parametrize("mutate", [
    lambda p, s: p[0]["records"][0].update(lazy_slot=5),          # slot out of range
    lambda p, s: p[0]["records"][0].update(power_slot=3),         # no such exponent
    lambda p, s: p[0]["records"][2].update(parent_slot=0),        # root with a parent
    lambda p, s: p[0]["records"][2].update(reads_register=False),  # parent never read
    lambda p, s: p[0]["records"][0].update(reads_register=True),  # reads an unwritten register
    lambda p, s: p[0]["records"][0].update(sub=0),                # root nested in itself
    lambda p, s: p[0]["records"][0].update(sub=7),                # no such program
    lambda p, s: s[0].insert(0, 1),                               # exponent set not ascending
    lambda p, s: p[0].update(root_child_ends=[2, 1]),             # ends not ascending
    lambda p, s: p[0].update(variable=1),                         # variable out of range
])
def test_malformed_programs_are_rejected(mutate):
    progs, sets = _horner_3x2_2x_1()
    mutate(progs, sets)
    with pytest.raises(ValueError):
        pe.CompiledProgram.from_compiled(progs, sets)


def test_nested_program_referenced_twice_is_rejected():
    inner = {"records": [{"coeff": 1.0, "lazy_slot": 0}], "register_count": 1, "variable": 1}
    root = {"records": [
        {"sub": 1, "power_slot": 0, "lazy_slot": 0, "parent_slot": 0},
        {"sub": 1, "lazy_slot": 0, "reads_register": True},
    ], "register_count": 1, "variable": 0}
    with pytest.raises(ValueError):
        pe.CompiledProgram.from_compiled([root, inner], [[1], []])


def test_register_check_clean_programs():
    # reference enable_register_check (eval.hpp:142-145): compiled programs
    # leave the register file clean
    for wl in (W.c2(1000, "estrin"), W.c3()):
        prog = pe.compile(wl.poly, wl.schemes)
        assert pe._lib.lib().pe_program_check_registers(prog.handle) == 0


def test_register_check_flags_unconsumed_value():
    # record 0 accumulates into register 1, which nothing reads: the walk
    # leaves a value behind (structurally valid for the lowering, unclean)
    progs = [{"records": [
        {"coeff": 3.0, "power_slot": 0, "lazy_slot": 0, "parent_slot": 0},
        {"coeff": 5.0, "lazy_slot": 1, "parent_slot": 1},
        {"coeff": 2.0, "power_slot": 0, "lazy_slot": 0, "parent_slot": 1,
         "reads_register": True},
        {"coeff": 1.0, "lazy_slot": 1, "reads_register": True},
    ], "register_count": 2, "variable": 0}]
    prog = pe.CompiledProgram.from_compiled(progs, [[1]])
    assert pe._lib.lib().pe_program_check_registers(prog.handle) == 0
    progs[0]["records"][3]["reads_register"] = False
    with pytest.raises(ValueError):  # rejected outright: register 1 never read
        pe.CompiledProgram.from_compiled(progs, [[1]])


def test_evaluate_parallel_validates_workers():
    wl = W.c2(1000, "estrin")
    prog = pe.compile(wl.poly, wl.schemes)
    ev = pe.Evaluator(pe.DoubleDomain(), prog)
    with pytest.raises(ValueError):
        ev.evaluate_parallel(wl.points(4), 0)
