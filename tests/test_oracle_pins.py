"""Pins of the oracle (oracle/) against what the paper and the mathematics fix.

Each test states what it pins: values PAPER.md prints (tests/golden/, with citations),
closed forms, invariants (Thm. 1 corner agreement, Thm. 4 certificate, multilinearity),
textbook / library routines (binomial distribution via scipy.stats), and brute force.
None of these re-types the oracle's own formula.
"""
from fractions import Fraction
from itertools import product

import numpy as np
import pytest
from scipy import stats

from conftest import golden, read_golden
from oracle import cdp, exact
from oracle.exact import OR, XOR, XNOR, CARD_GE, CARD_LE, NAE
from oracle.formula import OracleFormula, ParseError, parse
from oracle.philox import philox4x32_10, uniform_pm1
from oracle import solve as osolve
import synth

KINDS = [OR, XOR, XNOR, CARD_GE, CARD_LE, NAE]
F = Fraction


def _fr(tok):
    return Fraction(tok)


def _all_signatures(kmax):
    for k in range(1, kmax + 1):
        for kd in KINDS:
            bounds = range(0, k + 1) if kd in (CARD_GE, CARD_LE) else [0]
            for b in bounds:
                yield kd, k, b


# ---------------------------------------------------------------- T0: Walsh coefficients


def test_eq1_walsh_coefficients():
    """Eq. 1 in the paper's [e4..e0] order, by Thm. 1 literally and by the grouped form."""
    g = read_golden("eq1_card4_ge2_walsh.txt")
    want = [_fr(t) for t in g["coeffs"][0]]
    got_grouped = list(reversed(exact.walsh_coeffs(CARD_GE, 4, 2)))
    got_thm1 = list(reversed(exact.walsh_coeffs_thm1(CARD_GE, 4, 2)))
    assert got_grouped == want
    assert got_thm1 == want


def test_walsh_grouped_equals_thm1_bruteforce():
    """Hamming-weight grouping == literal Thm. 1 enumeration for every signature with k <= 7."""
    for kd, k, b in _all_signatures(7):
        assert list(exact.walsh_coeffs(kd, k, b)) == exact.walsh_coeffs_thm1(kd, k, b), (kd, k, b)


def test_xor_walsh_is_top_monomial():
    """App. B: f^_XOR = [1 0 ... 0] in [e_k..e_0] order; XNOR is its negation."""
    for k in range(1, 9):
        a = exact.walsh_coeffs(XOR, k, 0)
        assert a[k] == 1 and all(v == 0 for v in a[:k])
        assert list(exact.walsh_coeffs(XNOR, k, 0)) == [-v for v in a]


def test_esp_special_values():
    """Def. 2: esp(0..0) = [1,0..0]; esp(1,1,1,1) = binomials [1,4,6,4,1]."""
    assert exact.esp([0, 0, 0]) == [1, 0, 0, 0]
    assert exact.esp([1, 1, 1, 1]) == [1, 4, 6, 4, 1]


# ---------------------------------------------------------------- paper worked examples


@pytest.fixture(scope="module")
def eg3():
    vals = read_golden("eg2_eg3_values.txt")
    x = [_fr(t) for t in vals["x"][0]]
    return x, vals


def test_eg3_value_and_eg2_gradient_exact(eg3):
    """T0 exact: WE = -59/128 and grad (19/64,19/64,33/64,33/64)."""
    x, vals = eg3
    assert exact.fe_exact(CARD_GE, 2, x) == _fr(vals["value"][0][0])
    assert exact.grad_exact(CARD_GE, 2, x) == [_fr(t) for t in vals["grad"][0]]
    assert exact.fe_multilinear_bruteforce(CARD_GE, 2, x) == _fr(vals["value"][0][0])
    assert exact.grad_multilinear_bruteforce(CARD_GE, 2, x) == [_fr(t) for t in vals["grad"][0]]


def test_eg3_eg5_dp(eg3):
    """T2 DP: value, gradient and Eg. 5's P(true)/P(false)."""
    x, vals = eg3
    F = parse(open(golden("eg2_eg3_card4_ge2.hnf")).read())
    f, g = cdp.evaluate(F, np.array([[float(v) for v in x]]))
    assert abs(f[0] - float(_fr(vals["value"][0][0]))) < 1e-15
    np.testing.assert_allclose(g[0], [float(_fr(t)) for t in vals["grad"][0]], atol=1e-15, rtol=0)
    ptrue = float(_fr(vals["p_true"][0][0])); pfalse = float(_fr(vals["p_false"][0][0]))
    assert abs(f[0] - (pfalse - ptrue)) < 1e-15


def test_eg5_eg6_bdd_messages(eg3):
    """M_TD and M_BU at the BDD nodes (i literals seen, t True)."""
    x, _ = eg3
    q, beta = cdp.messages(CARD_GE, 2, [float(v) for v in x])
    msgs = read_golden("eg5_eg6_messages.txt")
    for i, t, v in msgs["M_TD"]:
        assert abs(q[int(i)][int(t)] - float(_fr(v))) < 1e-15
    for i, t, v in msgs["M_BU"]:
        psat = (1.0 - beta[int(i)][int(t)]) / 2.0
        assert abs(psat - float(_fr(v))) < 1e-15


def _poly2(c, x1, x2):
    return c[0] + c[1] * x1 + c[2] * x2 + c[3] * x1 * x2


def test_eg7_objective_and_saddle():
    """Eg. 7: F equals the printed polynomial; grad = 0 at the saddle; after the
    ERWA update w' = (0.6, 1) the gradient is (-2/15, 2/15) (reading #5)."""
    F = parse(open(golden("eg7_saddle.hnf")).read())
    vals = read_golden("eg7_values.txt")
    c = [float(_fr(t)) for t in vals["poly_F"][0]]
    rng = np.random.default_rng(1)
    X = rng.uniform(-1, 1, size=(50, 2))
    f, _ = cdp.evaluate(F, X)
    np.testing.assert_allclose(f, _poly2(c, X[:, 0], X[:, 1]), atol=1e-15)
    s = np.array([[float(_fr(t)) for t in vals["saddle"][0]]])
    _, g = cdp.evaluate(F, s)
    assert np.max(np.abs(g)) < 1e-15
    w = osolve.erwa_update(np.ones(2), np.array([0, 1]), 0.4)
    np.testing.assert_allclose(w, [float(_fr(t)) for t in vals["weights_after"][0]], rtol=0, atol=1e-15)
    ca = [float(_fr(t)) for t in vals["poly_F_after"][0]]
    fa, ga = cdp.evaluate_weighted(F, w, X)
    np.testing.assert_allclose(fa, _poly2(ca, X[:, 0], X[:, 1]), atol=1e-15)
    _, ga = cdp.evaluate_weighted(F, w, s)
    np.testing.assert_allclose(ga[0], [float(_fr(t)) for t in vals["grad_after"][0]], atol=1e-15)


def test_eg8_local_optimum():
    """Eg. 8: unsat pattern (0,1,0), ERWA weights (3/5,1,3/5), gradient (-3/5,-2/5,-2/5,-3/5)."""
    F = parse(open(golden("eg8_local.hnf")).read())
    vals = read_golden("eg8_values.txt")
    x = np.array([[float(v) for v in vals["x"][0]]])
    cnt, fw, U = cdp.check(F, x, want_U=True)
    assert list(U) == [int(v) for v in vals["unsat"][0]]
    assert cnt[0] == 1 and fw[0] == 1.0
    w = osolve.erwa_update(np.ones(3), U, 0.4)
    np.testing.assert_allclose(w, [float(_fr(t)) for t in vals["weights_after"][0]], atol=1e-15)
    _, g = cdp.evaluate_weighted(F, w, x)
    np.testing.assert_allclose(g[0], [float(_fr(t)) for t in vals["grad_after"][0]], atol=1e-15)
    # F = x1x2 + x2x3 + x3x4 at random points
    X = np.random.default_rng(2).uniform(-1, 1, size=(20, 4))
    f, _ = cdp.evaluate(F, X)
    np.testing.assert_allclose(f, X[:, 0] * X[:, 1] + X[:, 1] * X[:, 2] + X[:, 2] * X[:, 3], atol=1e-15)


def test_erwa_paper_values():
    """Prop. 3 with alpha = 0.4: r = 0 -> 0.6, r = 1 -> 1.0; max U = 0 skips."""
    w = osolve.erwa_update(np.ones(3), np.array([0, 5, 0]), 0.4)
    np.testing.assert_allclose(w, [0.6, 1.0, 0.6], atol=1e-16)
    assert np.array_equal(osolve.erwa_update(np.full(3, 0.3), np.zeros(3, np.int32), 0.4), np.full(3, 0.3))
    # geometric convergence |w_t - r| = (1-a)^t |w_0 - r|
    U = np.array([1])
    w = np.array([0.0])
    for t in range(1, 6):
        w = osolve.erwa_update(w, U, 0.4)
        assert abs(abs(w[0] - 1.0) - 0.6 ** t) < 1e-15


# ---------------------------------------------------------------- invariants, closed forms


def test_corners_equal_truth_values():
    """Thm. 1: FE = +-1 (the truth value) at every corner; all signatures k <= 9."""
    for kd, k, b in _all_signatures(9):
        C = np.array(list(product((1.0, -1.0), repeat=k)))
        for row in C:
            fe, _ = cdp.constraint(kd, b, row)
            t = int(np.sum(row < 0))
            assert fe == (-1.0 if exact.satisfied(kd, k, b, t) else 1.0), (kd, k, b, row)


def test_dp_matches_exact_tiers_small_k():
    """T2 (fp64 DP) vs T0 (exact Eq. 3) and T1 (brute-force multilinear) at random dyadic points."""
    rng = np.random.default_rng(5)
    for kd, k, b in _all_signatures(6):
        for _ in range(2):
            l = [F(int(v), 64) for v in rng.integers(-64, 65, size=k)]
            fe, dl = cdp.constraint(kd, b, [float(v) for v in l])
            fe0 = exact.fe_exact(kd, b, l)
            fe1 = exact.fe_multilinear_bruteforce(kd, b, l)
            assert fe0 == fe1
            assert abs(fe - float(fe0)) < 1e-15
            g0 = exact.grad_exact(kd, b, l)
            assert g0 == exact.grad_multilinear_bruteforce(kd, b, l)
            assert max(abs(a - float(c)) for a, c in zip(dl, g0)) < 1e-15


@pytest.mark.parametrize("k", [16, 32, 64])
def test_dp_matches_exact_rationals_medium_k(k):
    """T2 vs T0 exact rationals at k = 16/32/64 on uniform, near-corner and corner points (B4)."""
    rng = np.random.default_rng(k)
    for kd, b in [(CARD_LE, k // 4), (CARD_GE, k // 2), (OR, 0), (XOR, 0), (NAE, 0)]:
        for dist in ("U", "N", "C"):
            if dist == "U":
                l = [F(int(v), 1 << 20) for v in rng.integers(-(1 << 20), (1 << 20) + 1, size=k)]
            elif dist == "N":
                l = [F(int(s) * ((1 << 20) - int(d)), 1 << 20) for s, d in
                     zip(rng.choice([-1, 1], size=k), rng.integers(0, 1000, size=k))]
            else:
                l = [F(int(s)) for s in rng.choice([-1, 1], size=k)]
            fe, dl = cdp.constraint(kd, b, [float(v) for v in l])
            assert abs(fe - float(exact.fe_exact(kd, b, l))) < 1e-14
            if k <= 32:
                g0 = exact.grad_exact(kd, b, l)
                assert max(abs(a - float(c)) for a, c in zip(dl, g0)) < 1e-14


def test_closed_forms():
    """OR = 2 prod (1+l)/2 - 1; XOR = prod l; XNOR = -prod l; NAE = 2prod(1+l)/2 + 2prod(1-l)/2 - 1;
    AND (GE b=k) = 1 - 2 prod (1-l)/2; LE b=0 = 1 - 2 prod (1+l)/2 (SURVEY 8(c) special cases)."""
    rng = np.random.default_rng(9)
    for k in (1, 2, 3, 7, 20, 60):
        for _ in range(5):
            l = rng.uniform(-1, 1, size=k)
            A = np.prod((1 + l) / 2); Bp = np.prod((1 - l) / 2); X = np.prod(l)
            tol = 1e-14
            assert abs(cdp.constraint(OR, 0, l)[0] - (2 * A - 1)) < tol
            assert abs(cdp.constraint(XOR, 0, l)[0] - X) < tol
            assert abs(cdp.constraint(XNOR, 0, l)[0] + X) < tol
            assert abs(cdp.constraint(NAE, 0, l)[0] - (2 * A + 2 * Bp - 1)) < tol
            assert abs(cdp.constraint(CARD_GE, k, l)[0] - (1 - 2 * Bp)) < tol
            assert abs(cdp.constraint(CARD_LE, 0, l)[0] - (1 - 2 * A)) < tol
            # k = 1: OR = XOR = l
            if k == 1:
                assert abs(cdp.constraint(OR, 0, l)[0] - l[0]) < tol


@pytest.mark.parametrize("k", [500, 1237, 2000])
def test_long_constraints_binomial(k):
    """Equal literal values: T ~ Binomial(k, p) (textbook); two value groups: convolution of two
    binomial pmfs.  FE(CARD_LE b) = sum_t f(t) P(T=t) via scipy.stats (library routine)."""
    rng = np.random.default_rng(k)
    for b in (k // 4, k // 2, (3 * k) // 4):
        lv = rng.uniform(-0.9, 0.9)
        fe, dl = cdp.constraint(CARD_LE, b, np.full(k, lv))
        p = (1 - lv) / 2
        want = 1 - 2 * stats.binom.cdf(b, k, p)
        assert abs(fe - want) < 1e-12, (fe, want)
        # symmetric literals -> equal gradient components
        assert np.ptp(dl) < 1e-12
        # two groups
        k1 = k // 3
        la, lb = rng.uniform(-1, 1, size=2)
        l = np.concatenate([np.full(k1, la), np.full(k - k1, lb)])
        pmf = np.convolve(stats.binom.pmf(np.arange(k1 + 1), k1, (1 - la) / 2),
                          stats.binom.pmf(np.arange(k - k1 + 1), k - k1, (1 - lb) / 2))
        fvals = np.where(np.arange(k + 1) <= b, -1.0, 1.0)
        fe, _ = cdp.constraint(CARD_LE, b, l)
        assert abs(fe - float(np.dot(fvals, pmf))) < 1e-12


@pytest.mark.parametrize("k", [5, 64, 800])
def test_gradient_central_differences(k):
    """FE is affine in each l_i (Thm. 1), so the central difference with any h is exact up to
    rounding: (FE(l_i + h) - FE(l_i - h)) / 2h with h = 1/4 (S:188-196 idea)."""
    rng = np.random.default_rng(k + 1)
    for kd, b in [(CARD_GE, k // 3), (CARD_LE, k // 2), (NAE, 0), (OR, 0)]:
        l = rng.uniform(-0.7, 0.7, size=k)
        _, dl = cdp.constraint(kd, b, l)
        h = 0.25
        for i in rng.choice(k, size=min(k, 6), replace=False):
            lp = l.copy(); lp[i] += h
            lm = l.copy(); lm[i] -= h
            fd = (cdp.constraint(kd, b, lp)[0] - cdp.constraint(kd, b, lm)[0]) / (2 * h)
            assert abs(fd - dl[i]) < 1e-12


def test_range_bounds():
    """|FE| <= 1 and |dFE/dl| <= 1 on [-1,1]^k (multilinear range)."""
    rng = np.random.default_rng(3)
    for kd, k, b in _all_signatures(12):
        l = rng.uniform(-1, 1, size=k)
        fe, dl = cdp.constraint(kd, b, l)
        assert abs(fe) <= 1 + 1e-15 and np.max(np.abs(dl)) <= 1 + 1e-15


def test_formula_chain_rule_exact():
    """Whole-formula f and grad (Def. 3, Prop. 1) T2 vs T0 exact rationals, all kinds, weights."""
    inst = synth.random_mixed(n=12, m=30, seed=4, kmax=8)
    Fo = OracleFormula.from_arrays(*inst.arrays())
    x = synth.points("U", 3, inst.n, 11, np.float64)
    f, g = cdp.evaluate(Fo, x)
    for b in range(3):
        fe, ge = exact.formula_eval_exact(inst.n, list(Fo.constraints()), [F(float(v)) for v in x[b]])
        assert abs(f[b] - float(fe)) < 1e-13
        np.testing.assert_allclose(g[b], [float(v) for v in ge], atol=1e-13, rtol=0)


def test_certificate_thm4():
    """Thm. 4: at a satisfying corner f = -sum w; at any corner f = sum_c w_c (+-1) and the check
    count matches a direct truth-table count (brute force over all 2^n corners of a c1-shaped formula)."""
    inst = synth.config1(0)
    Fo = OracleFormula.from_arrays(*inst.arrays())
    n = inst.n
    # all corners of 20 vars is 1M points: sample 4096 corners + the brute-force satisfiable check below
    X = synth.points("C", 4096, n, 21, np.float64)
    f = cdp.evaluate(Fo, X, grad=False)
    cnt, fw = cdp.check(Fo, X)
    np.testing.assert_allclose(f, -Fo.m + 2 * cnt, atol=1e-12)
    # direct count
    for b in range(0, 4096, 512):
        c = 0
        for kd, bd, w, ls in Fo.constraints():
            t = sum(1 for l in ls if (X[b, abs(l) - 1] < 0) == (l > 0))
            c += not exact.satisfied(kd, len(ls), bd, t)
        assert c == cnt[b]


def test_bruteforce_c1_satisfiability():
    """Brute force over all 2^20 corners of c1 seed 0 (vectorised): oracle check agrees with numpy
    truth evaluation on the satisfying set; any zero-count corner gives f = -m (Thm. 4)."""
    inst = synth.config1(0)
    Fo = OracleFormula.from_arrays(*inst.arrays())
    n = inst.n
    ids = np.arange(1 << n, dtype=np.uint32)
    bits = ((ids[:, None] >> np.arange(n, dtype=np.uint32)) & 1).astype(bool)  # True = variable True
    lit = inst.lits.reshape(-1, 3)
    v = np.abs(lit) - 1
    val = bits[:, v] == (lit > 0)
    sat_all = val.any(axis=2).all(axis=1)
    sols = np.nonzero(sat_all)[0]
    if len(sols):
        x = np.where(bits[sols[:8]], -1.0, 1.0)
        cnt, _ = cdp.check(Fo, x)
        assert np.all(cnt == 0)
        f = cdp.evaluate(Fo, x, grad=False)
        np.testing.assert_allclose(f, -Fo.m, atol=1e-12)
    nons = np.nonzero(~sat_all)[0][:8]
    cnt, _ = cdp.check(Fo, np.where(bits[nons], -1.0, 1.0))
    assert np.all(cnt > 0)


def test_tie_rule_zero_is_false():
    """sgn(0) = False (reading #10): OR(x1) at x1 = 0 and -0.0 is unsatisfied; OR(-x1) satisfied."""
    Fo = OracleFormula.from_constraints(1, [(OR, 0, 1.0, [1])])
    cnt, _ = cdp.check(Fo, np.array([[0.0], [-0.0], [-1e-300]]))
    assert list(cnt) == [1, 1, 0]
    Fn = OracleFormula.from_constraints(1, [(OR, 0, 1.0, [-1])])
    cnt, _ = cdp.check(Fn, np.array([[0.0], [-0.0]]))
    assert list(cnt) == [0, 0]


# ---------------------------------------------------------------- parser, RNG, solve


def test_parser_errors():
    for bad in ["p hnf 2 1\no 1 3 0\n", "p hnf 2 1\no 1 1 0\n", "p hnf 3 1\nd 4 1 2 3 0\n",
                "p hnf 2 1\no 1 2\n", "o 1 0\n", "p hnf 2 1\nq 1 0\n", "p hnf 2 1\no 0\n"]:
        with pytest.raises(ParseError):
            parse(bad)
    Fo = parse("c x\np whnf 3 2\n2.5 x 1 -2 0\n0.5 a 1 1 2 3 0\n")
    assert list(Fo.kind) == [XOR, CARD_LE] and list(Fo.weight) == [2.5, 0.5] and list(Fo.bound) == [0, 1]


def test_philox_known_answers():
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    for line in open(golden("philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        t = [int(v, 16) for v in line.split()]
        assert philox4x32_10(t[0:4], t[4:6]) == tuple(t[6:10])
    u = uniform_pm1(123, 7, 0, 1000)
    assert min(u) > -1 and max(u) < 1 and abs(np.mean(u)) < 0.1


def test_oracle_solve_semantics():
    """Alg. 1 on tiny formulas: Eg. 7's formula is SAT (verified); {x1, not x1} is UNKNOWN;
    PGD iterates stay in the box and accepted f is non-increasing."""
    F7 = parse(open(golden("eg7_saddle.hnf")).read())
    sat, x, _ = osolve.cls_solve(F7, B=4, seed=1, max_rounds=5, P=osolve.Params(max_inner=50))
    assert sat and cdp.check(F7, x[None])[0][0] == 0
    Fu = OracleFormula.from_constraints(1, [(OR, 0, 1.0, [1]), (OR, 0, 1.0, [-1])])
    sat, _, _ = osolve.cls_solve(Fu, B=4, seed=1, max_rounds=3, P=osolve.Params(max_inner=30))
    assert not sat
    inst = synth.config1(3)
    Fo = OracleFormula.from_arrays(*inst.arrays())
    P = osolve.Params(max_inner=40)
    st = osolve.State(x=osolve.initial_points(5, range(8), Fo.n), f=None, g=None, eta=None, done=None,
                      iters=None, w=np.ones(Fo.m))
    osolve.start_round(Fo, st, P)
    prev = st.f.copy()
    for _ in range(40):
        osolve.pgd_iteration(Fo, st, P)
        assert np.all(st.x <= 1) and np.all(st.x >= -1)
        assert np.all(st.f <= prev + 1e-12)
        prev = st.f.copy()


# ---- solve-loop pins written out by hand (rephase and the PGD eta schedule were unpinned)

def _saddle_formula():
    """f(x) = x1 x2 + x1/4 + x2/4: XOR(x1, x2) has FE = l1 l2 (t odd <=> l1 l2 = -1 at the corners, Thm. 1) and a
    unit clause (x) has FE = x (OR with k = 1, 2 (1+x)/2 - 1), weighted 1/4 each (Def. 3)."""
    return OracleFormula.from_constraints(2, [(XOR, 0, 1.0, [1, 2]), (OR, 0, 0.25, [1]), (OR, 0, 0.25, [2])])


def test_pgd_eta_schedule_hand_derived():
    """Alg. 4 in the monotone projected-Armijo reading (#16), worked by hand with dyadic
    numbers (exact in fp64), under the formula's static weights.  From x = (0, 0): g = (x2 + 1/4, x1 + 1/4) = (1/4, 1/4), eta0 = 4, c1 = 1e-4.
      1. x' = (-1, -1): f' = 1 - 1/2 = 1/2 > f + c1 <g, x'-x> = -5e-5          reject, eta 4 -> 2
      2. x' = (-1/2, -1/2): f' = 1/4 - 1/4 = 0 > -2.5e-5                       reject, eta 2 -> 1
      3. x' = (-1/4, -1/4): f' = 1/16 - 1/8 = -1/16 <= -1.25e-5                accept, eta -> min(2, 4) = 2
      4. g(-1/4, -1/4) = (0, 0): x' = x, f' = f <= f + 0                       accept, eta -> 4
    max_inner = 4 then marks the point done: a 5th iteration changes nothing.  With eta_min = 1.5 instead, the
    second rejection leaves eta = 1 < eta_min and the point is done after iteration 2."""
    F = _saddle_formula()
    f0, g0 = cdp.evaluate(F, np.zeros((1, 2)))
    assert f0[0] == 0.0 and np.array_equal(g0[0], [0.25, 0.25])
    P = osolve.Params(eta0=4.0, max_inner=4, adaptive_weights=False)
    st = osolve.State(x=np.zeros((1, 2)), f=None, g=None, eta=None, done=None, iters=None, w=F.weight.copy())
    osolve.start_round(F, st, P)
    want = [(False, 2.0, (0.0, 0.0), 0.0), (False, 1.0, (0.0, 0.0), 0.0), (True, 2.0, (-0.25, -0.25), -0.0625),
            (True, 4.0, (-0.25, -0.25), -0.0625)]
    for acc_w, eta_w, x_w, f_w in want:
        _, _, _, acc = osolve.pgd_iteration(F, st, P)
        assert bool(acc[0]) == acc_w and st.eta[0] == eta_w
        assert np.array_equal(st.x[0], x_w) and st.f[0] == f_w
    assert st.done[0] and st.iters[0] == 4
    osolve.pgd_iteration(F, st, P)
    assert st.eta[0] == 4.0 and np.array_equal(st.x[0], [-0.25, -0.25]) and st.iters[0] == 4
    P2 = osolve.Params(eta0=4.0, eta_min=1.5, max_inner=100, adaptive_weights=False)
    st = osolve.State(x=np.zeros((1, 2)), f=None, g=None, eta=None, done=None, iters=None, w=F.weight.copy())
    osolve.start_round(F, st, P2)
    osolve.pgd_iteration(F, st, P2)
    assert not st.done[0] and st.eta[0] == 2.0
    osolve.pgd_iteration(F, st, P2)
    assert st.done[0] and st.eta[0] == 1.0
    osolve.pgd_iteration(F, st, P2)
    assert st.eta[0] == 1.0 and np.array_equal(st.x[0], [0.0, 0.0])


def test_pgd_projection_arc_armijo():
    """The sufficient-decrease test uses the PROJECTED step x' - x (the projection arc), not -eta g: from x = (-1, 1)
    on f = x1 x2 + x1/4 + x2/4, g = (5/4, -3/4); eta = 1 gives x - g = (-9/4, 7/4), clipped to (-1, 1) = x itself, so
    x' - x = 0, f' = f and the step is accepted with eta -> min(2, eta0) (with -eta g it would need f' <= f - 2.125e-4
    and be rejected)."""
    F = _saddle_formula()
    P = osolve.Params(eta0=1.0, max_inner=10, adaptive_weights=False)
    st = osolve.State(x=np.array([[-1.0, 1.0]]), f=None, g=None, eta=None, done=None, iters=None, w=F.weight.copy())
    osolve.start_round(F, st, P)
    assert np.array_equal(st.g[0], [1.25, -0.75]) and st.f[0] == -1.0
    xp, fp, _, acc = osolve.pgd_iteration(F, st, P)
    assert np.array_equal(xp[0], [-1.0, 1.0]) and fp[0] == -1.0 and bool(acc[0]) and st.eta[0] == 1.0


def test_rephase_phases_hand_derived():
    """O / F / R of P:611-615 in the (ROF)^inf cycle, staggered by global point index (reading #20): at new
    round r the point with global index b takes phase "ROF"[(r - 1 + b) mod 3] -- O keeps x, F is exactly -x, R is a
    fresh uniform draw of the stream (seed, b, r) (Alg. 1 line 1's sampler, keyed by the NEW round)."""
    n, seed = 6, 31
    x = np.array([[0.5, -0.25, 0.125, -1.0, 1.0, 0.0]] * 6) * np.arange(1, 7)[:, None] / 6
    P = osolve.Params(policy="ROF")
    # point0 = 0, round 1: b = 0 R, 1 O, 2 F, 3 R, 4 O, 5 F
    y = osolve.rephase(x, seed, 0, 1, P)
    assert np.array_equal(y[1], x[1]) and np.array_equal(y[4], x[4])
    assert np.array_equal(y[2], -x[2]) and np.array_equal(y[5], -x[5])
    assert np.array_equal(y[0], uniform_pm1(seed, 0, 1, n)) and np.array_equal(y[3], uniform_pm1(seed, 3, 1, n))
    assert not np.array_equal(y[0], uniform_pm1(seed, 0, 0, n))          # the new round's stream, not round 0's
    # point0 = 5, round 2: global b = 5..10, (1 + b) mod 3 = 0, 1, 2, 0, 1, 2 -> R O F R O F
    y = osolve.rephase(x, seed, 5, 2, P)
    assert np.array_equal(y[0], uniform_pm1(seed, 5, 2, n)) and np.array_equal(y[3], uniform_pm1(seed, 8, 2, n))
    assert np.array_equal(y[1], x[1]) and np.array_equal(y[2], -x[2]) and np.array_equal(y[5], -x[5])
    # (RF)^inf: b even -> R at odd rounds; R only: every point redrawn
    y = osolve.rephase(x, seed, 0, 1, osolve.Params(policy="RF"))
    assert np.array_equal(y[0], uniform_pm1(seed, 0, 1, n)) and np.array_equal(y[1], -x[1])
    y = osolve.rephase(x, seed, 0, 3, osolve.Params(policy="R"))
    assert all(np.array_equal(y[i], uniform_pm1(seed, i, 3, n)) for i in range(6))


def test_fista_schedule_hand_derived():
    """The FISTA reading (#16b; P:939 names jaxopt's accelerated projected gradient) worked by hand on
    f = x1 x2 + x1/4 + x2/4 from x = (0, 0), eta0 = 4, with dyadic values (exact in fp64):
      y = (0, 0), f_y = 0, g_y = (1/4, 1/4)
      1. x+ = (-1, -1): f+ = 1/2 > f_y + <g_y, x+ - y> + |x+ - y|^2 / 8 = -1/2 + 1/4 = -1/4        reject, eta -> 2
      2. x+ = (-1/2, -1/2): f+ = 0 > -1/4 + 1/8 = -1/8                                              reject, eta -> 1
      3. x+ = (-1/4, -1/4): f+ = -1/16 <= -1/8 + 1/16 = -1/16 (equality)                             accept, t: 1 -> (1 + 5^.5) / 2,
         beta = 0, so y = x+ (its f and gradient (0, 0) are at hand), eta -> 2, next trial x+ = y
      4. x+ = y: f+ = f_y <= f_y                                                                     accept, beta = (t - 1) / t' != 0:
         the next evaluation is y' = x + beta (x - x_prev) = x (x_prev = x): phase 0
      5. the y evaluation: f_y = -1/16, g_y = 0; the next trial is x+ = y."""
    F = _saddle_formula()
    P = osolve.Params(eta0=4.0, max_inner=50, adaptive_weights=False)
    st = osolve.fista_start_round(F, np.zeros((1, 2)), F.weight.copy(), P)
    assert np.array_equal(st.xp[0], [-1.0, -1.0]) and st.phase[0] == 1
    want = [("reject", 2.0, (-0.5, -0.5)), ("reject", 1.0, (-0.25, -0.25)), ("accept", 2.0, (-0.25, -0.25)),
            ("accept", 4.0, (-0.25, -0.25)), ("y", 4.0, (-0.25, -0.25))]
    for k, (act_w, eta_w, xp_w) in enumerate(want):
        acts = osolve.fista_iteration(F, st, P)
        assert acts[0] == act_w and st.eta[0] == eta_w and np.array_equal(st.xp[0], xp_w), k
    assert np.array_equal(st.x[0], [-0.25, -0.25]) and st.f[0] == -0.0625
    assert abs(st.t[0] - (1 + np.sqrt(1 + 4 * ((1 + 5 ** 0.5) / 2) ** 2)) / 2) < 1e-15
    assert st.iters[0] == 5 and st.phase[0] == 1


def test_fista_descends_and_stays_feasible():
    """On a random 3-SAT instance every accepted x stays in the box (trials are projected; only the extrapolation
    points y may leave it) and after 60 evaluations the accepted f is below the start for every point."""
    inst = synth.config1(3)
    Fo = OracleFormula.from_arrays(*inst.arrays())
    P = osolve.Params(eta0=8.0, max_inner=60)
    st = osolve.fista_start_round(Fo, osolve.initial_points(5, range(8), Fo.n), np.ones(Fo.m), P)
    f0 = st.f.copy()
    for _ in range(60):
        osolve.fista_iteration(Fo, st, P)
        assert np.all(np.abs(st.x) <= 1)
    assert np.all(st.f <= f0 + 1e-12) and np.mean(st.f) < np.mean(f0)
