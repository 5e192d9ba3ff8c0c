"""SURVEY 8(f) f3, host side: the planted Max-Cut generator and the relative score."""
import itertools

import numpy as np

import synth
from oracle import cdp
from oracle.formula import OracleFormula
from paper_2308_15020_b200.maxsat import relative_score


def test_planted_maxcut_structure():
    inst = synth.planted_maxcut(4, 5, seed=3)
    u, v, w, cl = (inst.meta[k] for k in ("edges_u", "edges_v", "edges_w", "cluster"))
    assert inst.n == 20 and inst.m == len(u) and np.all(u < v)
    assert np.all(w == np.where(cl[u] == cl[v], 1.0, 2.0))
    assert np.all(inst.kind == synth.XOR) and np.array_equal(np.diff(inst.offsets), np.full(inst.m, 2))
    # about half of the C(n, 2) pairs
    assert 0.35 < inst.m / (20 * 19 / 2) < 0.65


def test_falsified_weight_is_uncut_weight():
    """The XOR encoding: the oracle's falsified static weight of any bipartition equals the uncut edge weight."""
    inst = synth.planted_maxcut(3, 4, seed=1)
    Fo = OracleFormula.from_arrays(*inst.arrays())
    u, v, w = (inst.meta[k] for k in ("edges_u", "edges_v", "edges_w"))
    rng = np.random.default_rng(0)
    X = np.where(rng.random((50, inst.n)) < 0.5, -1.0, 1.0)
    _, fw = cdp.check(Fo, X)
    uncut = np.array([w[(x[u] < 0) == (x[v] < 0)].sum() for x in X])
    assert np.allclose(fw, uncut)


def test_relative_score_examples():
    # SPEC S:466-468 examples
    costs = {"A": 8.0, "B": 10.0, "C": 8.0}
    assert relative_score(costs, "A") == 1.0 and relative_score(costs, "C") == 1.0
    assert abs(relative_score(costs, "B") - 1.0 / 3.0) < 1e-15
    assert relative_score({"A": 5.0, "B": 5.0}, "B") == 1.0
    assert relative_score({"A": 7.0}, "A") == 1.0


def brute_force_min_uncut(inst):
    Fo = OracleFormula.from_arrays(*inst.arrays())
    X = np.array(list(itertools.product((-1.0, 1.0), repeat=inst.n)))
    _, fw = cdp.check(Fo, X)
    return float(fw.min())


def test_brute_force_reference_small():
    inst = synth.planted_maxcut(2, 4, seed=0)
    assert brute_force_min_uncut(inst) <= np.sum(inst.weight)
