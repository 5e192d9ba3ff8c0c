"""Weighted MaxSAT / optimisation mode (PAPER.md Benchmark 3).

For optimisation Thm. 4 gives no certificate, so the CLS loop runs with fixed weights and the
(RF)^inf rephasing policy and keeps an incumbent: the rounded point of minimum falsified
weight.  The falsified weight of a corner a = sgn(x) comes from one batched evaluation of f at the corners:
f(a) = sum_c w_c FE_c(a) = -W + 2 * falsified(a) (FE = -1 on satisfied, +1 on falsified constraints, Thm. 1),
so falsified(a) = (f(a) + W) / 2 -- every step runs in libffsat's kernels; torch only rounds and takes the argmin.
"""
from __future__ import annotations

import time

import numpy as np


def relative_score(costs: dict, solver) -> float:
    """score(s, i) = (max_s cost - cost_s + 1) / (max_s cost - min_s cost + 1), cost = falsified weight."""
    vals = list(costs.values())
    hi, lo = max(vals), min(vals)
    return (hi - costs[solver] + 1.0) / (hi - lo + 1.0)


def solve_maxsat(ctx, batch: int = 32, rounds: int = 100, seed: int = 0, max_inner: int = 100, timeout_s: float = 0.0):
    """Batched CLS in optimisation mode on a loaded Context (device).  Returns (best falsified weight, assignment
    int8 [n] -1 True / +1 False, rounds run, seconds)."""
    import torch

    t0 = time.perf_counter()
    weights = ctx.export()[2]
    W = float(np.sum(weights))
    s = ctx.search(batch, seed=seed, max_inner=max_inner, check_every=max_inner, policy="RF", adaptive_weights=0)
    T = s.tensors()
    best_w, best_a = np.inf, None
    r = 0
    for r in range(1, rounds + 1):
        s.begin_round()
        s.iterate(max_inner)
        corners = torch.where(T["x"] < 0, -1.0, 1.0).to(T["x"].dtype)
        f, _, _ = ctx.eval(corners, grad=False)
        fw = (f + W) * 0.5
        i = int(torch.argmin(fw).item())
        if float(fw[i].item()) < best_w:
            best_w = float(fw[i].item())
            best_a = np.where(corners[i].cpu().numpy() < 0, -1, 1).astype(np.int8)
        if timeout_s > 0 and time.perf_counter() - t0 > timeout_s:
            break
        s.restart()
    # exact host re-check of the incumbent (integer count and weight)
    n_unsat, fw_exact = ctx.check(best_a)
    return fw_exact, best_a, r, time.perf_counter() - t0
