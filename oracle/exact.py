"""oracle/exact.py -- TEST INFRASTRUCTURE ONLY (tiers T0 and T1 of the oracle).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs
may import this module.  It shares no code with the CUDA product path.

Everything here is exact rational arithmetic (``fractions.Fraction``) written
straight from the paper's definitions:

* truth_by_count      -- constraint semantics by the number t of True literals
                         (-1 = True; readings #11, #12).
* walsh_coeffs_thm1   -- Thm. 1 literally: f^(S) = 2^-n sum_x f(x) prod_{i in S} x_i,
                         enumerated over all 2^k corners (k <= 12).
* walsh_coeffs        -- the same sum grouped by Hamming weight (symmetric constraint,
                         P:116-118): f^_j = 2^-k sum_t f(t) sum_u (-1)^u C(j,u) C(k-j,t-u).
                         (This is the corrected form of SPEC's S:137, reading #6.)
* esp                 -- elementary symmetric polynomials (Def. 2) via the
                         convolution esp = [x1,1]*...*[xk,1] (Eq. 6).
* fe_exact            -- WE_c(x) = f^_c . esp(x) (Eq. 3).
* grad_exact          -- dFE/dl_i by the exact multilinear difference
                         (FE(l_i=1) - FE(l_i=-1)) / 2 (FE is affine in each l_i, Thm. 1).
* fe_multilinear_bruteforce / grad_multilinear_bruteforce -- T1: the multilinear
                         extension sum_y f(#{y=-1}) prod_i (1 + l_i y_i)/2 over all 2^k corners.
"""
from __future__ import annotations

from fractions import Fraction
from functools import lru_cache
from itertools import product
from math import comb

OR, XOR, XNOR, CARD_GE, CARD_LE, NAE = 0, 1, 2, 3, 4, 5
KIND_NAMES = {OR: "OR", XOR: "XOR", XNOR: "XNOR", CARD_GE: "CARD_GE", CARD_LE: "CARD_LE", NAE: "NAE"}


def satisfied(kind: int, k: int, bound: int, t: int) -> bool:
    """Constraint satisfied by a corner with t True literals."""
    if kind == OR:
        return t >= 1
    if kind == XOR:
        return t % 2 == 1
    if kind == XNOR:
        return t % 2 == 0
    if kind == CARD_GE:
        return t >= bound
    if kind == CARD_LE:
        return t <= bound
    if kind == NAE:
        return 0 < t < k
    raise ValueError(kind)


def truth_by_count(kind: int, k: int, bound: int = 0) -> list[int]:
    """f(t) in {+1,-1}; -1 = satisfied."""
    return [-1 if satisfied(kind, k, bound, t) else 1 for t in range(k + 1)]


def walsh_coeffs_thm1(kind: int, k: int, bound: int = 0) -> list[Fraction]:
    """Thm. 1 by brute force over all 2^k corners; returns [f^_0 .. f^_k]
    where f^_j = f^(S) for S = {1..j} (any S of size j, by symmetry)."""
    if k > 14:
        raise ValueError("brute force Thm. 1 limited to k <= 14")
    out = []
    for j in range(k + 1):
        s = 0
        for y in product((1, -1), repeat=k):
            t = sum(1 for yi in y if yi == -1)
            fy = -1 if satisfied(kind, k, bound, t) else 1
            mono = 1
            for i in range(j):
                mono *= y[i]
            s += fy * mono
        out.append(Fraction(s, 2 ** k))
    return out


@lru_cache(maxsize=None)
def walsh_coeffs(kind: int, k: int, bound: int = 0) -> tuple:
    """Thm. 1 grouped by Hamming weight: corners with t Trues of which u lie in S (|S| = j)
    number C(j,u) C(k-j,t-u) and give prod_{i in S} x_i = (-1)^u."""
    f = truth_by_count(kind, k, bound)
    out = []
    for j in range(k + 1):
        s = 0
        for t in range(k + 1):
            kt = 0
            for u in range(0, min(j, t) + 1):
                if t - u <= k - j:
                    kt += (-1) ** u * comb(j, u) * comb(k - j, t - u)
            s += f[t] * kt
        out.append(Fraction(s, 2 ** k))
    return tuple(out)


def esp(ls) -> list[Fraction]:
    """[e_0 .. e_k] of the values ls by the convolution of Eq. 6."""
    e = [Fraction(1)]
    for x in ls:
        x = Fraction(x)
        nxt = [Fraction(0)] * (len(e) + 1)
        for j, ej in enumerate(e):
            nxt[j] += ej          # the '1' entry of [x, 1]
            nxt[j + 1] += ej * x  # the 'x' entry of [x, 1]
        e = nxt
    return e


def fe_exact(kind: int, bound: int, ls) -> Fraction:
    """WE_c = sum_j f^_j e_j(l) (Eq. 3)."""
    k = len(ls)
    a = walsh_coeffs(kind, k, bound)
    e = esp(ls)
    return sum((aj * ej for aj, ej in zip(a, e)), Fraction(0))


def grad_exact(kind: int, bound: int, ls) -> list[Fraction]:
    """dFE/dl_i = (FE(l_i = 1) - FE(l_i = -1)) / 2, exact because FE is multilinear."""
    ls = [Fraction(v) for v in ls]
    out = []
    for i in range(len(ls)):
        hi = list(ls); hi[i] = Fraction(1)
        lo = list(ls); lo[i] = Fraction(-1)
        out.append((fe_exact(kind, bound, hi) - fe_exact(kind, bound, lo)) / 2)
    return out


def fe_multilinear_bruteforce(kind: int, bound: int, ls, exact: bool = True):
    """T1: FE(l) = sum_{y in {+-1}^k} f(#{y_i=-1}) prod_i (1 + l_i y_i)/2."""
    k = len(ls)
    one = Fraction(1) if exact else 1.0
    half = Fraction(1, 2) if exact else 0.5
    vals = [Fraction(v) if exact else float(v) for v in ls]
    s = 0 * one
    for y in product((1, -1), repeat=k):
        t = sum(1 for yi in y if yi == -1)
        fy = -1 if satisfied(kind, k, bound, t) else 1
        p = one
        for li, yi in zip(vals, y):
            p *= (one + li * yi) * half
        s += fy * p
    return s


def grad_multilinear_bruteforce(kind: int, bound: int, ls, exact: bool = True):
    """T1 gradient: dFE/dl_i = sum_y f(y) (y_i/2) prod_{j != i} (1 + l_j y_j)/2."""
    k = len(ls)
    one = Fraction(1) if exact else 1.0
    half = Fraction(1, 2) if exact else 0.5
    vals = [Fraction(v) if exact else float(v) for v in ls]
    out = []
    for i in range(k):
        s = 0 * one
        for y in product((1, -1), repeat=k):
            t = sum(1 for yi in y if yi == -1)
            fy = -1 if satisfied(kind, k, bound, t) else 1
            p = y[i] * half
            for j, (lj, yj) in enumerate(zip(vals, y)):
                if j != i:
                    p *= (one + lj * yj) * half
            s += fy * p
        out.append(s)
    return out


def formula_eval_exact(n: int, cons, x):
    """f and grad of a whole formula (Def. 3, Eq. 5; chain rule Prop. 1) in exact rationals.
    cons: list of (kind, bound, weight, lits) with DIMACS lits."""
    x = [Fraction(v) for v in x]
    f = Fraction(0)
    g = [Fraction(0)] * n
    for kind, bound, w, lits in cons:
        w = Fraction(w)
        ls = [x[abs(l) - 1] if l > 0 else -x[abs(l) - 1] for l in lits]
        f += w * fe_exact(kind, bound, ls)
        for l, d in zip(lits, grad_exact(kind, bound, ls)):
            g[abs(l) - 1] += w * (d if l > 0 else -d)
    return f, g
