"""oracle/solve.py -- TEST INFRASTRUCTURE ONLY: the CLS loop semantics in plain fp64 numpy.

Follows PAPER.md's Alg. 1, Alg. 4 projected gradient descent,
the ERWA weighting of Prop. 3 (alpha = 0.4 P:988/P:1138) and the O/F/R
rephasing policy ((ROF)^inf P:1013/P:1145), in the readings DESIGN.md
lists (#15 ERWA w0 = 1 and skip when max U = 0; #16 monotone projected Armijo
backtracking with one trial per iteration; #10 sgn(0) = False; #20 phase offset =
global point index).  f and grad come from the T2 DP (oracle/dp.c).

Per point b, one PGD iteration:
    x'   = clip(x - eta * g, -1, 1)                               (Alg. 4 lines 2-3)
    f',g'= f(x'), grad f(x') under the current weights w
    accept iff f' <= f + c1 * <g, x' - x>                          (Armijo on the projection arc)
    accept: x, f, g <- x', f', g';  eta <- min(2 eta, eta0)
    reject: eta <- eta / 2
    done  iff eta < eta_min or iterations == max_inner
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import cdp
from .formula import OracleFormula
from .philox import uniform_pm1


@dataclass
class Params:
    eta0: float = 1.0
    eta_min: float = 1e-12
    armijo_c1: float = 1e-4
    alpha: float = 0.4
    max_inner: int = 500
    policy: str = "ROF"
    adaptive_weights: bool = True


@dataclass
class State:
    x: np.ndarray            # [B][n]
    f: np.ndarray            # [B]
    g: np.ndarray            # [B][n]
    eta: np.ndarray          # [B]
    done: np.ndarray         # [B] bool
    iters: np.ndarray        # [B] int
    w: np.ndarray            # [m]
    rnd: int = 0
    point0: int = 0          # global index of local point 0 (restart sharding)
    log: list = field(default_factory=list)


def initial_points(seed: int, points, n: int, rnd: int = 0) -> np.ndarray:
    """Alg. 1 line 1: x0 sampled uniformly from [-1,1]^n, one Philox stream per global point."""
    return np.array([uniform_pm1(seed, int(b), rnd, n) for b in points], dtype=np.float64).reshape(len(points), n)


def start_round(F: OracleFormula, st: State, P: Params):
    st.f, st.g = cdp.evaluate_weighted(F, st.w, st.x)
    st.eta = np.full(len(st.f), P.eta0)
    st.done = np.zeros(len(st.f), dtype=bool)
    st.iters = np.zeros(len(st.f), dtype=np.int64)


def pgd_iteration(F: OracleFormula, st: State, P: Params):
    """One trial step for every not-done point (Alg. 4)."""
    act = ~st.done
    xp = np.clip(st.x - st.eta[:, None] * st.g, -1.0, 1.0)
    xp[~act] = st.x[~act]
    fp, gp = cdp.evaluate_weighted(F, st.w, xp)
    d = np.einsum("bn,bn->b", st.g, xp - st.x)
    acc = act & (fp <= st.f + P.armijo_c1 * d)
    rej = act & ~acc
    st.x[acc] = xp[acc]; st.f[acc] = fp[acc]; st.g[acc] = gp[acc]
    st.eta[acc] = np.minimum(2.0 * st.eta[acc], P.eta0)
    st.eta[rej] = 0.5 * st.eta[rej]
    st.iters[act] += 1
    st.done |= act & ((st.eta < P.eta_min) | (st.iters >= P.max_inner))
    return xp, fp, gp, acc


# ---- accelerated projected gradient (FISTA, Beck & Teboulle 2009) with backtracking: the paper's solver runs
#      jaxopt's projected gradient with FISTA acceleration and a line search; reading #16b.
#      Per point, one evaluation per iteration, a two-phase machine:
#        phase 1 (a trial x+ = clip(y - eta g_y) was evaluated): accept iff f(x+) <= f(y) + <g_y, x+ - y>
#                 + |x+ - y|^2 / (2 eta) (the quadratic upper bound); accept: x_prev, x <- x, x+; t <- (1 +
#                 sqrt(1 + 4 t^2)) / 2, beta = (t_old - 1) / t; eta <- min(2 eta, eta0); if beta = 0 the new y is
#                 x+ itself (its f, g are at hand) and the next trial is proposed, else the next evaluation is
#                 y = x + beta (x - x_prev) (phase 0); reject: eta <- eta / 2, next trial from the same y.
#        phase 0 (y was evaluated): f_y, g_y <- f(y), grad f(y); the next trial is proposed (phase 1).
#      Every evaluation counts as an iteration; done at eta < eta_min or max_inner iterations.


@dataclass
class FistaState:
    x: np.ndarray            # [B][n] accepted x_k
    f: np.ndarray            # f(x_k)
    g: np.ndarray            # grad f(x_k)
    xm: np.ndarray           # x_{k-1}
    y: np.ndarray            # current extrapolation point
    fy: np.ndarray
    gy: np.ndarray
    xp: np.ndarray           # the next point to evaluate
    t: np.ndarray
    eta: np.ndarray
    phase: np.ndarray        # 1: xp is a trial from y; 0: xp is the next y
    done: np.ndarray
    iters: np.ndarray
    w: np.ndarray


def fista_propose(st: FistaState, b: int):
    st.xp[b] = np.clip(st.y[b] - st.eta[b] * st.gy[b], -1.0, 1.0)
    st.phase[b] = 1


def fista_start_round(F: OracleFormula, x: np.ndarray, w: np.ndarray, P: Params) -> FistaState:
    f, g = cdp.evaluate_weighted(F, w, x)
    B = len(f)
    st = FistaState(x=x.copy(), f=f, g=g, xm=x.copy(), y=x.copy(), fy=f.copy(), gy=g.copy(), xp=x.copy(),
                    t=np.ones(B), eta=np.full(B, P.eta0), phase=np.ones(B, np.int64), done=np.zeros(B, bool),
                    iters=np.zeros(B, np.int64), w=w)
    for b in range(B):
        fista_propose(st, b)
    return st


def fista_iteration(F: OracleFormula, st: FistaState, P: Params):
    """One evaluation for every point, then each point's phase step (see above).  Returns per-point actions:
    'y' (phase 0 consumed), 'accept', 'reject', or None (done)."""
    fp, gp = cdp.evaluate_weighted(F, st.w, st.xp)
    acts = []
    for b in range(len(fp)):
        if st.done[b]:
            acts.append(None)
            continue
        if st.phase[b] == 0:
            st.y[b], st.fy[b], st.gy[b] = st.xp[b], fp[b], gp[b]
            fista_propose(st, b)
            acts.append("y")
        else:
            dx = st.xp[b] - st.y[b]
            q = st.fy[b] + np.dot(st.gy[b], dx) + np.dot(dx, dx) / (2.0 * st.eta[b])
            if fp[b] <= q:
                st.xm[b], st.x[b], st.f[b], st.g[b] = st.x[b].copy(), st.xp[b].copy(), fp[b], gp[b]
                t_new = (1.0 + np.sqrt(1.0 + 4.0 * st.t[b] ** 2)) / 2.0
                beta = (st.t[b] - 1.0) / t_new
                st.t[b] = t_new
                st.eta[b] = min(2.0 * st.eta[b], P.eta0)
                if beta == 0.0:
                    st.y[b], st.fy[b], st.gy[b] = st.x[b].copy(), fp[b], gp[b]
                    fista_propose(st, b)
                else:
                    st.xp[b] = st.x[b] + beta * (st.x[b] - st.xm[b])
                    st.phase[b] = 0
                acts.append("accept")
            else:
                st.eta[b] = 0.5 * st.eta[b]
                fista_propose(st, b)
                acts.append("reject")
        st.iters[b] += 1
        if st.eta[b] < P.eta_min or st.iters[b] >= P.max_inner:
            st.done[b] = True
    return acts


def erwa_update(w: np.ndarray, U: np.ndarray, alpha: float) -> np.ndarray:
    """Prop. 3: w <- (1-alpha) w + alpha r, r_c = U_c / max U; skipped when max U = 0."""
    mx = int(U.max()) if len(U) else 0
    if mx == 0:
        return w.copy()
    r = U.astype(np.float64) / mx
    return (1.0 - alpha) * w + alpha * r


def rephase(x: np.ndarray, seed: int, point0: int, new_round: int, P: Params) -> np.ndarray:
    """O (keep) / F (negate) / R (fresh Philox uniform) per point; phase index (round-1 + global b) mod len(policy)."""
    out = x.copy()
    L = len(P.policy)
    for i in range(x.shape[0]):
        b = point0 + i
        ph = P.policy[(new_round - 1 + b) % L]
        if ph == "F":
            out[i] = -x[i]
        elif ph == "R":
            out[i] = np.array(uniform_pm1(seed, b, new_round, x.shape[1]))
    return out


def cls_solve(F: OracleFormula, B: int, seed: int, max_rounds: int, P: Params = Params()):
    """Small-scale Alg. 1 with p_t = B points.  Returns (sat, assignment_x or None, rounds)."""
    x = initial_points(seed, range(B), F.n)
    st = State(x=x, f=None, g=None, eta=None, done=None, iters=None, w=np.ones(F.m))
    for rnd in range(max_rounds):
        st.rnd = rnd
        start_round(F, st, P)
        while not st.done.all():
            pgd_iteration(F, st, P)
        cnt, _, U = cdp.check(F, st.x, want_U=True)
        hit = np.nonzero(cnt == 0)[0]
        if len(hit):
            return True, st.x[hit[0]].copy(), rnd + 1
        if P.adaptive_weights:
            st.w = erwa_update(st.w, U, P.alpha)
        st.x = rephase(st.x, seed, 0, rnd + 1, P)
    return False, None, max_rounds
