"""Polynomial and point text formats of the reference CLI.

Restates the reference grammar (proj/core/src/parser.cpp:27-186):

    poly   := [sign] term { ('+' | '-') term }
    term   := integer | integer '*' factors | factors
    factors:= factor { '*' factor }
    factor := ident [ '^' natural ]          ident = alpha (alnum | '_')*

Variables are discovered in order of first appearance unless an explicit
order is given; repeated factors add exponents; terms are canonicalised by the
native front-end. Points use `name=value` bindings separated by commas
(parser.cpp:324-360); interval values are `[lo,hi]`.

Errors carry the 0-based character position like the reference's ParseError.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .api import Polynomial


class ParseError(ValueError):
    def __init__(self, message: str, position: int):
        super().__init__(f"{message} (at position {position})")
        self.position = position


class BindingError(ValueError):
    pass


@dataclass
class _Term:
    coefficient: int
    exponents: dict


class _Parser:
    def __init__(self, text: str, variables=None):
        self.t = text
        self.pos = 0
        self.fixed = variables is not None
        self.vars = list(variables) if variables is not None else []

    def at_end(self):
        return self.pos >= len(self.t)

    def peek(self):
        return self.t[self.pos]

    def skip(self):
        while not self.at_end() and self.peek().isspace():
            self.pos += 1

    def integer(self):
        self.skip()
        s = self.pos
        while not self.at_end() and self.peek().isdigit():
            self.pos += 1
        if s == self.pos:
            raise ParseError("expected an integer", self.pos)
        return int(self.t[s:self.pos])

    def natural(self):
        self.skip()
        s = self.pos
        while not self.at_end() and self.peek().isdigit():
            self.pos += 1
        if s == self.pos:
            raise ParseError("exponent must be a natural number", self.pos)
        v = int(self.t[s:self.pos])
        if v >= 2**32:
            raise ParseError("exponent out of range", s)
        return v

    def slot(self, name, at):
        if name in self.vars:
            return self.vars.index(name)
        if self.fixed:
            raise ParseError(f"unknown variable '{name}'", at)
        self.vars.append(name)
        return len(self.vars) - 1

    def factor(self, term):
        self.skip()
        s = self.pos
        if self.at_end() or not self.peek().isalpha():
            raise ParseError("expected a variable name", self.pos)
        self.pos += 1
        while not self.at_end() and (self.peek().isalnum() or self.peek() == "_"):
            self.pos += 1
        name = self.t[s:self.pos]
        e = 1
        self.skip()
        if not self.at_end() and self.peek() == "^":
            self.pos += 1
            e = self.natural()
        v = self.slot(name, s)
        term.exponents[v] = term.exponents.get(v, 0) + e

    def term(self, sign):
        self.skip()
        if self.at_end():
            raise ParseError("expected a term", self.pos)
        term = _Term(1, {})
        if self.peek().isdigit():
            term.coefficient = self.integer()
        elif self.peek().isalpha():
            self.factor(term)
        else:
            raise ParseError(f"unexpected character '{self.peek()}'", self.pos)
        self.skip()
        while not self.at_end() and self.peek() == "*":
            self.pos += 1
            self.factor(term)
            self.skip()
        if sign < 0:
            term.coefficient = -term.coefficient
        return term

    def parse(self):
        self.skip()
        if self.at_end():
            raise ParseError("empty polynomial expression", self.pos)
        sign = 1
        if self.peek() in "+-":
            sign = -1 if self.peek() == "-" else 1
            self.pos += 1
        terms = [self.term(sign)]
        self.skip()
        while not self.at_end():
            c = self.peek()
            if c not in "+-":
                raise ParseError(f"expected '+' or '-' before '{c}'", self.pos)
            self.pos += 1
            terms.append(self.term(-1 if c == "-" else 1))
            self.skip()
        return terms


def parse_polynomial(text: str, variables=None) -> Polynomial:
    """Parses the reference grammar into a Polynomial with int64 coefficients
    (ValueError if a merged coefficient does not fit int64)."""
    p = _Parser(text, variables)
    terms = p.parse()
    nv = max(1, len(p.vars))
    names = tuple(p.vars) if p.vars else ("x",)
    exps = np.zeros((len(terms), nv), dtype=np.uint32)
    coefs = []
    for i, t in enumerate(terms):
        for v, e in t.exponents.items():
            exps[i, v] = e
        coefs.append(t.coefficient)
    if any(c < -(2**63) or c >= 2**63 for c in coefs):
        raise ParseError("coefficient does not fit int64 (BigInt is out of scope on the GPU)", 0)
    return Polynomial(exps, np.array(coefs, dtype=np.int64), names)


def parse_point(text: str, variables, domain: str):
    """`x=1.5, y=[0.5,0.75]` -> per-variable values in variable order
    (reference parse_point, parser.cpp:324-360)."""
    values = [None] * len(variables)
    if text.strip():
        parts, depth, cur = [], 0, ""
        for ch in text:
            if ch == "[":
                depth += 1
            elif ch == "]":
                depth -= 1
            if ch == "," and depth == 0:
                parts.append(cur)
                cur = ""
            else:
                cur += ch
        parts.append(cur)
        for b in parts:
            b = b.strip()
            if not b:
                raise BindingError("empty binding")
            if "=" not in b:
                raise BindingError(f"binding is missing '=': '{b}'")
            name, val = (s.strip() for s in b.split("=", 1))
            if name not in variables:
                raise BindingError(f"unknown variable '{name}' in point")
            k = list(variables).index(name)
            if values[k] is not None:
                raise BindingError(f"variable '{name}' bound twice")
            values[k] = _scalar(val, domain)
    for i, v in enumerate(values):
        if v is None:
            raise BindingError(f"variable '{variables[i]}' is unbound")
    return values


def _scalar(text, domain):
    try:
        if domain == "int":
            return int(text)
        if domain == "float":
            return float(text)
        if domain == "interval":
            t = text.strip()
            if t.startswith("[") and t.endswith("]"):
                lo, hi = (float(s) for s in t[1:-1].split(","))
            else:
                lo = hi = float(t)
            if not lo <= hi:
                raise BindingError(f"invalid interval '{text}'")
            return (lo, hi)
    except (TypeError, ValueError) as e:
        if isinstance(e, BindingError):
            raise
        raise BindingError(f"malformed {domain} literal: '{text}'") from None
    raise BindingError(f"unknown domain '{domain}'")
