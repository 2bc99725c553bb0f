"""`python -m paper_1307_5655_b200 {compile,eval,bench}` — GPU batch CLI.

Mirrors the reference CLI (proj/tools/main.cpp:123-356): same subcommands,
scheme grammar (`name` | `upper:lower@N`, one scheme applied to every
variable), output formats (shortest round-trip doubles, `[lo,hi]` intervals)
and exit codes (main.cpp:32-36): 0 ok, 1 parse error, 2 unknown scheme,
3 binding/domain error, 4 I/O error. New relative to the reference:
`eval --points FILE [--out FILE]` evaluates a whole batch (.npy of shape
(n, nvars) — (n, nvars, 2) for intervals — or .csv) on the GPU, and `bench`
times batch throughput; its CSV keeps the reference header
(bench.cpp:189-200) with median_ns = nanoseconds per point.
"""
from __future__ import annotations

import argparse
import csv
import os
import sys
import time

import numpy as np

from . import api as pe
from .parser import BindingError, ParseError, parse_point, parse_polynomial

EXIT_OK, EXIT_PARSE, EXIT_SCHEME, EXIT_BINDING, EXIT_IO = 0, 1, 2, 3, 4


class UnknownScheme(Exception):
    pass


class IoError(Exception):
    pass


def _scheme(name: str):
    try:
        return pe.scheme_from_name(name)
    except (KeyError, ValueError):
        raise UnknownScheme(f"unknown scheme '{name}'") from None


def _fmt(x: float) -> str:
    r = repr(float(x))
    return r[:-2] if r.endswith(".0") else r


def _compile(poly_text, scheme_name, var_order="", as_float=False):
    variables = [v for v in var_order.split(",") if v] if var_order else None
    p = parse_polynomial(poly_text, variables)
    if as_float:
        p = pe.Polynomial(p.exponents, p.coefficients.astype(np.float64), p.variables)
    s = _scheme(scheme_name)
    return p, pe.compile(p, [s] * p.nvars)


def cmd_compile(a):
    p, prog = _compile(a.poly, a.scheme, a.vars)
    if a.dot:
        try:
            with open(a.dot, "w") as f:
                f.write(prog.dot())
        except OSError as e:
            raise IoError(f"cannot open '{a.dot}' for writing: {e}") from None
    if a.stats:
        # reference main.cpp:139-148: root-tree node count, maxima over nested trees
        inf = prog.info()
        sets = [prog.exponent_set(v) for v in range(p.nvars)]
        print(f"nodes: {len(prog.records())}")
        print(f"max_partial_degree: {max((max(s) for s in sets if s), default=0)}")
        print(f"max_lazy_height: {inf['max_registers'] - 1}")
        for v, name in enumerate(p.variables):
            print(f"exponents[{name}]: {len(prog.exponent_set(v))}")
    return EXIT_OK


def _domain(name, strict=False):
    if name == "int":
        return pe.BigIntDomain()
    if name == "float":
        return pe.DoubleDomain(strict=strict)
    if name == "interval":
        return pe.IntervalDomain()
    raise BindingError(f"unknown domain '{name}'")


def _load_points(path, nvars, interval):
    try:
        if path.endswith(".npy"):
            arr = np.load(path)
        else:
            with open(path) as f:
                rows = [r for r in csv.reader(f) if r]
            if rows and any(not _is_num(c) for c in rows[0]):
                rows = rows[1:]
            arr = np.array([[float(c) for c in r] for r in rows])
            if interval:
                arr = arr.reshape(len(arr), -1, 2)
    except (OSError, ValueError) as e:
        raise IoError(f"cannot read points from '{path}': {e}") from None
    want = (nvars, 2) if interval else (nvars,)
    if arr.ndim != 1 + len(want) or tuple(arr.shape[1:]) != want:
        raise BindingError(f"points must have shape (n, {', '.join(map(str, want))}), got {arr.shape}")
    return arr


def _is_num(s):
    try:
        float(s)
        return True
    except ValueError:
        return False


def cmd_eval(a):
    p, prog = _compile(a.poly, a.scheme, a.vars, as_float=a.domain != "int")
    dom = _domain(a.domain, a.strict)
    ev = pe.Evaluator(dom, prog, device=a.device)
    if a.points:
        arr = _load_points(a.points, p.nvars, a.domain == "interval")
        if a.domain == "int":
            res = ev.evaluate([np.ascontiguousarray(arr[:, v], dtype=np.int64) for v in range(p.nvars)])
            out = np.asarray(res)
        elif a.domain == "float":
            out = np.asarray(ev.evaluate([arr[:, v] for v in range(p.nvars)]))
        else:
            lo, hi = ev.evaluate(([arr[:, v, 0] for v in range(p.nvars)],
                                  [arr[:, v, 1] for v in range(p.nvars)]))
            out = np.stack([lo, hi], axis=1)
        if a.out:
            try:
                if a.out.endswith(".npy"):
                    np.save(a.out, out)
                else:
                    with open(a.out, "w") as f:
                        for row in np.atleast_2d(out.T).T:
                            f.write(",".join(str(int(v)) if a.domain == "int" else _fmt(v)
                                             for v in np.atleast_1d(row)) + "\n")
            except OSError as e:
                raise IoError(f"cannot write '{a.out}': {e}") from None
        else:
            for row in out:
                print(_row(row, a.domain))
        return EXIT_OK
    vals = parse_point(a.at or "", list(p.variables), a.domain)
    if a.domain == "int":
        r = ev.evaluate([np.array([v], dtype=np.int64) for v in vals])[0]
        print(int(r))
    elif a.domain == "float":
        print(_fmt(ev.evaluate([np.array([v]) for v in vals])[0]))
    else:
        lo, hi = ev.evaluate(([np.array([v[0]]) for v in vals], [np.array([v[1]]) for v in vals]))
        print(f"[{_fmt(lo[0])},{_fmt(hi[0])}]")
    return EXIT_OK


def _row(row, domain):
    if domain == "int":
        return str(int(row))
    if domain == "float":
        return _fmt(row)
    return f"[{_fmt(row[0])},{_fmt(row[1])}]"


def _degrees(text):
    if ":" in text:
        parts = [int(x) for x in text.split(":")]
        start, stop = parts[0], parts[1]
        step = parts[2] if len(parts) > 2 else 1
        if step <= 0:
            raise BindingError("expected start:stop[:step]")
        return list(range(start, stop + 1, step))
    return [int(x) for x in text.split(",") if x]


def cmd_bench(a):
    """Batch throughput per (degree, scheme) on dense random polynomials;
    reference CSV header, median_ns = ns per point over --reps timed batches."""
    import torch
    schemes = [_scheme(s) for s in a.schemes.split(",") if s]
    rng = np.random.Generator(np.random.PCG64(a.seed))
    dev = torch.device("cuda", max(a.device, 0))
    records = []
    for d in _degrees(a.degrees):
        c = rng.integers(-(2 ** (a.coeff_bits - 1)), 2 ** (a.coeff_bits - 1), d + 1)
        c[c == 0] = 1
        integer = a.domain == "int"
        poly = pe.Polynomial(np.arange(d, -1, -1).reshape(-1, 1),
                             c.astype(np.int64) if integer else c.astype(np.float64))
        if integer:
            x = torch.from_numpy(rng.integers(-1, 2, a.points)).to(dev)
        else:
            x = torch.from_numpy(rng.uniform(-1, 1, a.points)).to(dev)
        times = {}
        for s in schemes:
            prog = pe.compile(poly, [s])
            ev = pe.Evaluator(pe.BigIntDomain() if integer else pe.DoubleDomain(), prog,
                              deferred_checks=integer)
            out = ev.evaluate([x])
            samples = []
            for _ in range(a.reps):
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record()
                ev.evaluate([x], out=out)
                t1.record()
                torch.cuda.synchronize()
                samples.append(t0.elapsed_time(t1) * 1e6 / a.points)
            if integer:
                ev.synchronize()
            times[s.name] = float(np.median(samples))
        base = times.get("balanced")
        for name, ns in times.items():
            records.append((name, d, d + 1, a.coeff_bits, a.point_bits, 1, a.reps, ns,
                            ns / base if base else float("nan")))
    records.sort(key=lambda r: (r[1], r[0], r[5]))
    header = "scheme,degree,terms,coeff_bits,point_bits,workers,reps,median_ns,ratio_vs_balanced"
    lines = [header] + [f"{r[0]},{r[1]},{r[2]},{r[3]},{r[4]},{r[5]},{r[6]},{r[7]:.4f},{r[8]:.4f}"
                        for r in records]
    if a.csv:
        try:
            with open(a.csv, "w") as f:
                f.write("\n".join(lines) + "\n")
        except OSError as e:
            raise IoError(f"cannot open '{a.csv}' for writing: {e}") from None
    for r in records:
        print(f"degree {r[1]} ({r[2]} terms): {r[0]} {r[7]:.4f} ns/point [{r[8]:.4f}]")
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="polyeval-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("compile")
    c.add_argument("--poly", required=True)
    c.add_argument("--scheme", default="balanced")
    c.add_argument("--vars", default="")
    c.add_argument("--dot", default="")
    c.add_argument("--stats", action="store_true")
    e = sub.add_parser("eval")
    e.add_argument("--poly", required=True)
    e.add_argument("--scheme", default="balanced")
    e.add_argument("--vars", default="")
    e.add_argument("--domain", default="int", choices=["int", "float", "interval"])
    e.add_argument("--at", default="")
    e.add_argument("--points", default="")
    e.add_argument("--out", default="")
    e.add_argument("--strict", action="store_true", help="fp64: reference op order, bit-exact")
    e.add_argument("--device", type=int, default=-1)
    b = sub.add_parser("bench")
    b.add_argument("--schemes", default="horner,estrin,balanced")
    b.add_argument("--degrees", default="100,1000")
    b.add_argument("--points", type=int, default=1_000_000)
    b.add_argument("--domain", default="float", choices=["int", "float"])
    b.add_argument("--coeff-bits", type=int, default=8)
    b.add_argument("--point-bits", type=int, default=53)
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--csv", default="")
    b.add_argument("--device", type=int, default=-1)
    a = ap.parse_args(argv)
    try:
        return {"compile": cmd_compile, "eval": cmd_eval, "bench": cmd_bench}[a.cmd](a)
    except ParseError as ex:
        print(f"parse error: {ex}", file=sys.stderr)
        return EXIT_PARSE
    except UnknownScheme as ex:
        print(f"error: {ex}", file=sys.stderr)
        return EXIT_SCHEME
    except IoError as ex:
        print(f"I/O error: {ex}", file=sys.stderr)
        return EXIT_IO
    except (BindingError, ValueError, OverflowError) as ex:
        print(f"error: {ex}", file=sys.stderr)
        return EXIT_BINDING


if __name__ == "__main__":
    sys.exit(main())
