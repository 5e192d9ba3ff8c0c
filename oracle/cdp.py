"""oracle/cdp.py -- TEST INFRASTRUCTURE ONLY: ctypes access to oracle/dp.c (tier T2).

Builds oracle/liboracle.so with gcc on first use if it is missing (plain C, -O2,
OpenMP over points).  Only tests/, __graft_entry__ and bench.py's cpu_baseline /
reference legs may import this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .formula import OracleFormula

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dp.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.oracle_eval.argtypes = [ctypes.c_int32, ctypes.c_int64, P, P, P, P, P, ctypes.c_int64, P, P, P, ctypes.c_int]
        L.oracle_eval.restype = ctypes.c_int
        L.oracle_check.argtypes = [ctypes.c_int32, ctypes.c_int64, P, P, P, P, P, ctypes.c_int64, P, P, P, P]
        L.oracle_check.restype = ctypes.c_int
        L.oracle_constraint.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P]
        L.oracle_constraint.restype = ctypes.c_double
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_messages.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P]
        L.oracle_messages.restype = None
        _lib = L
    return _lib


def messages(kind: int, bound: int, l):
    """(q, beta) as lists of rows: q[i][t] = M_TD, beta[i][t] = expected truth value (Eg. 5/6)."""
    l = np.ascontiguousarray(l, dtype=np.float64)
    k = len(l)
    size = (k + 1) * (k + 2) // 2
    q = np.zeros(size); be = np.zeros(size)
    lib().oracle_messages(int(kind), k, int(bound), _p(l), _p(q), _p(be))
    rows = lambda a: [a[i * (i + 1) // 2: i * (i + 1) // 2 + i + 1] for i in range(k + 1)]
    return rows(q), rows(be)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def constraint(kind: int, bound: int, l):
    """FE and dFE/dl of one constraint at literal values l (fp64)."""
    l = np.ascontiguousarray(l, dtype=np.float64)
    dl = np.zeros_like(l)
    fe = lib().oracle_constraint(int(kind), len(l), int(bound), _p(l), _p(dl))
    return fe, dl


def evaluate(F: OracleFormula, x, grad: bool = True, threads: int = 0):
    """f[B], grad[B][n] at points x[B][n] (any float dtype, promoted exactly to fp64)."""
    x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
    B = x.shape[0]
    assert x.shape[1] == F.n
    f = np.zeros(B)
    g = np.zeros((B, F.n)) if grad else None
    lib().oracle_eval(F.n, F.m, _p(F.kind), _p(F.bound), _p(F.weight), _p(F.offsets), _p(F.lits),
                      B, _p(x), _p(f), _p(g), int(threads))
    return (f, g) if grad else f


def evaluate_weighted(F: OracleFormula, w, x, grad: bool = True, threads: int = 0):
    """As evaluate() with per-constraint weights w replacing F.weight (ERWA weights)."""
    G = OracleFormula(F.n, F.kind, F.bound, np.ascontiguousarray(w, dtype=np.float64), F.offsets, F.lits)
    return evaluate(G, x, grad, threads)


def check(F: OracleFormula, x, want_U: bool = False):
    """n_unsat[B], falsified_weight[B] (static weights) and optionally U[m] for sgn(x)."""
    x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
    B = x.shape[0]
    cnt = np.zeros(B, dtype=np.int64)
    fw = np.zeros(B)
    U = np.zeros(F.m, dtype=np.int32) if want_U else None
    lib().oracle_check(F.n, F.m, _p(F.kind), _p(F.bound), _p(F.weight), _p(F.offsets), _p(F.lits),
                       B, _p(x), _p(cnt), _p(fw), _p(U))
    return (cnt, fw, U) if want_U else (cnt, fw)


def max_threads() -> int:
    return int(lib().oracle_max_threads())
