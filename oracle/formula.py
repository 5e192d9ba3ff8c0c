"""oracle/formula.py -- TEST INFRASTRUCTURE ONLY.

The oracle's own reader for the hybrid formula text formats (SPEC S:99-104 grammar,
plus this build's extension `a <b> <lits> 0` = at-most-b and `n <lits> 0` = NAE,
DESIGN.md reading #12) and its array form.  Independent of the product's C++ parser
(paper_2308_15020_b200/csrc/host.cpp); parity tests feed the same file to both.

Array form (also what synth/ generators emit):
    kind    uint8[m]   0 OR, 1 XOR (odd), 2 XNOR (even), 3 CARD_GE, 4 CARD_LE, 5 NAE
    bound   int32[m]   the cardinality bound (GE/LE), else 0
    weight  float64[m]
    offsets int64[m+1]
    lits    int32[L]   DIMACS literals (1-based; negative = negated)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .exact import OR, XOR, XNOR, CARD_GE, CARD_LE, NAE


@dataclass
class OracleFormula:
    n: int
    kind: np.ndarray
    bound: np.ndarray
    weight: np.ndarray
    offsets: np.ndarray
    lits: np.ndarray

    @property
    def m(self) -> int:
        return int(len(self.kind))

    def constraints(self):
        for c in range(self.m):
            lo, hi = int(self.offsets[c]), int(self.offsets[c + 1])
            yield int(self.kind[c]), int(self.bound[c]), float(self.weight[c]), [int(v) for v in self.lits[lo:hi]]

    @staticmethod
    def from_arrays(n, kind, bound, weight, offsets, lits) -> "OracleFormula":
        m = len(kind)
        return OracleFormula(
            int(n),
            np.ascontiguousarray(kind, dtype=np.uint8),
            np.ascontiguousarray(bound if bound is not None else np.zeros(m), dtype=np.int32),
            np.ascontiguousarray(weight if weight is not None else np.ones(m), dtype=np.float64),
            np.ascontiguousarray(offsets, dtype=np.int64),
            np.ascontiguousarray(lits, dtype=np.int32),
        )

    @staticmethod
    def from_constraints(n, cons) -> "OracleFormula":
        kind, bound, weight, offs, lits = [], [], [], [0], []
        for kd, b, w, ls in cons:
            kind.append(kd); bound.append(b); weight.append(w)
            lits.extend(ls); offs.append(len(lits))
        return OracleFormula.from_arrays(n, kind, bound, weight, offs, lits)


class ParseError(ValueError):
    pass


def parse(text: str) -> OracleFormula:
    n = None
    weighted = False
    cons = []
    for lineno, raw in enumerate(text.splitlines(), 1):
        toks = raw.split()
        if not toks or toks[0] == "c":
            continue
        if toks[0] == "p":
            if len(toks) != 4 or toks[1] not in ("cnf", "hnf", "whnf"):
                raise ParseError(f"line {lineno}: bad header")
            fmt = toks[1]
            weighted = fmt == "whnf"
            n = int(toks[2])
            continue
        if n is None:
            raise ParseError(f"line {lineno}: constraint before header")
        w = 1.0
        if weighted:
            w = float(toks[0]); toks = toks[1:]
        if fmt == "cnf":
            kd, b, body = OR, 0, toks
        else:
            tag = toks[0]
            if tag == "o":
                kd, b, body = OR, 0, toks[1:]
            elif tag == "x":
                kd, b, body = XOR, 0, toks[1:]
            elif tag == "xn":
                kd, b, body = XNOR, 0, toks[1:]
            elif tag == "d":
                kd, b, body = CARD_GE, int(toks[1]), toks[2:]
            elif tag == "a":
                kd, b, body = CARD_LE, int(toks[1]), toks[2:]
            elif tag == "n":
                kd, b, body = NAE, 0, toks[1:]
            else:
                raise ParseError(f"line {lineno}: unknown constraint tag {tag!r}")
        if not body or body[-1] != "0":
            raise ParseError(f"line {lineno}: constraint not 0-terminated")
        ls = [int(t) for t in body[:-1]]
        if not ls:
            raise ParseError(f"line {lineno}: empty constraint")
        vs = [abs(l) for l in ls]
        if any(v < 1 or v > n for v in vs):
            raise ParseError(f"line {lineno}: literal out of range")
        if len(set(vs)) != len(vs):
            raise ParseError(f"line {lineno}: duplicate variable")
        if kd in (CARD_GE, CARD_LE) and not (0 <= b <= len(ls)):
            raise ParseError(f"line {lineno}: bound out of range")
        cons.append((kd, b, w, ls))
    if n is None:
        raise ParseError("missing header")
    return OracleFormula.from_constraints(n, cons)
