"""Multi-GPU host logic on CPU: world-size-2 gloo process groups.

The library's kernels need a GPU, so the per-rank compute here is the oracle (tests may use it): an
oracle-backed evaluator for constraint sharding and an oracle-backed search double for restart sharding.
What is under test is paper_2308_15020_b200/dist.py: the partitions, the collectives and the claim that a
restart-sharded run is identical to the single-process run of the same global points (F7)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_15020_b200 import dist as D
import synth
from oracle import cdp
from oracle import solve as osolve
from oracle.formula import OracleFormula


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)


# ---------------------------------------------------------------------------------------------- partitions


def test_point_ranges_partition():
    for B in (0, 1, 7, 32, 1000):
        for world in (1, 2, 3, 8):
            rs = [D.point_range(B, world, r) for r in range(world)]
            assert rs[0][0] == 0
            for (p0, b), (p1, _) in zip(rs, rs[1:]):
                assert p0 + b == p1
            assert sum(b for _, b in rs) == B
            assert max(b for _, b in rs) - min(b for _, b in rs) <= 1


def test_constraint_ranges_cover_and_balance():
    inst = synth.config3(0, n=600, m3=300, n_card=6, kmin=100, kmax=300)
    cost = D.constraint_cost(inst.kind, inst.bound, inst.offsets)
    assert np.all(cost[inst.kind == 0] == 3)            # clauses: k
    assert np.all(cost[inst.kind == 4] > 1000)          # long at-most: 12 k M'
    for world in (1, 2, 4):
        rs = D.constraint_ranges(inst.kind, inst.bound, inst.offsets, world)
        assert rs[0][0] == 0 and rs[-1][1] == inst.m
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        shares = [cost[c0:c1].sum() for c0, c1 in rs]
        assert max(shares) <= cost.sum() / world + cost.max()


def test_sub_formulas_sum_to_the_formula():
    inst = synth.random_mixed(n=40, m=120, seed=5, kmax=20)
    X = synth.points("U", 6, inst.n, 9, np.float64)
    f_full, g_full = cdp.evaluate(OracleFormula.from_arrays(*inst.arrays()), X)
    f, g = np.zeros_like(f_full), np.zeros_like(g_full)
    for c0, c1 in D.constraint_ranges(inst.kind, inst.bound, inst.offsets, 3):
        fs, gs = cdp.evaluate(OracleFormula.from_arrays(*D.sub_formula(*inst.arrays(), c0, c1)), X)
        f += fs
        g += gs
    assert np.allclose(f, f_full, rtol=0, atol=1e-12) and np.allclose(g, g_full, rtol=0, atol=1e-12)


# ---------------------------------------------------------------------------------------------- constraint sharding


def _sharded_eval_worker(rank, world, port, out):
    _init(rank, world, port)
    inst = synth.random_mixed(n=30, m=90, seed=21, kmax=16)
    X = synth.points("U", 5, inst.n, 3, np.float64)

    def evaluate(x):
        Fo = OracleFormula.from_arrays(*se.arrays)
        f, g = cdp.evaluate(Fo, x)
        u, _ = cdp.check(Fo, x)
        return torch.from_numpy(f), torch.from_numpy(g), torch.from_numpy(u.astype(np.int32))

    se = D.ShardedEval(inst.arrays(), rank, world, evaluate=evaluate)
    f, g, u = se.eval(X)
    # the overlapped variant (row blocks, asynchronous all-reduce of block i during block i + 1): the same bits
    f2, g2, u2 = se.eval(torch.from_numpy(X), chunks=2)
    same = bool(torch.equal(f2, f) and torch.equal(g2, g) and torch.equal(u2, u))
    if rank == 0:
        np.savez(out, f=f.numpy(), g=g.numpy(), u=u.numpy(), r=np.array(se.range), same=same)
    dist.destroy_process_group()


def test_constraint_sharded_eval_gloo(tmp_path):
    out = str(tmp_path / "se.npz")
    mp.spawn(_sharded_eval_worker, args=(2, free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    inst = synth.random_mixed(n=30, m=90, seed=21, kmax=16)
    X = synth.points("U", 5, inst.n, 3, np.float64)
    Fo = OracleFormula.from_arrays(*inst.arrays())
    f, g = cdp.evaluate(Fo, X)
    u, _ = cdp.check(Fo, X)
    assert 0 < r["r"][1] < inst.m                     # rank 0 holds a proper part
    assert np.allclose(r["f"], f, rtol=0, atol=1e-12)
    assert np.allclose(r["g"], g, rtol=0, atol=1e-12)
    assert np.array_equal(r["u"], u)
    assert bool(r["same"])


# ---------------------------------------------------------------------------------------------- restart sharding


class OracleSearch:
    """Test double of libffsat's Search on the oracle (oracle/solve.py semantics, fp64, CPU tensors).  Its reduce()
    mirrors ffsat_search_reduce's documented keys (include/ffsat.h) so dist.py's collectives can be tested on CPU."""

    def __init__(self, F, B, seed, point0, params):
        self.F, self.B, self.seed, self.point0, self.P = F, B, seed, point0, params
        self.st = osolve.State(x=osolve.initial_points(seed, range(point0, point0 + B), F.n), f=None, g=None,
                               eta=None, done=None, iters=None, w=np.ones(F.m), point0=point0)
        self.unsat = np.zeros(B, np.int32)
        self.U = np.zeros(F.m, np.int32)
        self.keys = np.zeros(2, np.int64)
        self.solved = np.zeros(B, np.int32)
        self.sol = np.zeros((B, F.n), np.int8)
        self.rnd = 0

    def tensors(self):
        return {"x": torch.from_numpy(self.st.x), "unsat": torch.from_numpy(self.unsat), "U": torch.from_numpy(self.U),
                "keys": torch.from_numpy(self.keys), "solved": torch.from_numpy(self.solved)}

    def begin_round(self):
        osolve.start_round(self.F, self.st, self.P)

    def iterate(self, n):
        for _ in range(n):
            osolve.pgd_iteration(self.F, self.st, self.P)

    def check(self):
        cnt, _, U = cdp.check(self.F, self.st.x, want_U=True)
        self.unsat[:] = cnt
        self.U[:] = U
        for b in np.nonzero((cnt == 0) & (self.solved == 0))[0]:
            self.solved[b] = 1
            self.sol[b] = np.where(self.st.x[b] < 0, -1, 1)

    def reduce(self):
        sol = np.nonzero(self.solved)[0]
        self.keys[0] = self.point0 + sol[0] if len(sol) else D.INT64_MAX
        self.keys[1] = min((int(u) << 32) | (self.point0 + b) for b, u in enumerate(self.unsat))

    def restart(self, U_global):
        if self.P.adaptive_weights:
            self.st.w = osolve.erwa_update(self.st.w, np.asarray(U_global), self.P.alpha)
        self.rnd += 1
        self.st.x[:] = osolve.rephase(self.st.x, self.seed, self.point0, self.rnd, self.P)

    def assignment(self, lp):
        if self.solved[lp]:
            return self.sol[lp].copy()
        return np.where(self.st.x[lp] < 0, -1, 1).astype(np.int8)


def _run_restart_sharded(rank, world, B_total, rounds, round_len):
    inst = synth.config1(4)
    Fo = OracleFormula.from_arrays(*inst.arrays())
    point0, B = D.point_range(B_total, world, rank)
    s = OracleSearch(Fo, B, 1234, point0, osolve.Params(max_inner=round_len))
    rs = D.RestartSharded(s, round_len, rank, world)
    rs.begin()
    keys = []
    for i in range(rounds * round_len):
        k = rs.step(i)
        if k is not None:
            keys.append([int(v) for v in k])
    cnt, gp, a = rs.incumbent()
    return point0, s.st.x.copy(), s.st.w.copy(), keys, (cnt, gp, a)


def _restart_worker(rank, world, port, out, B_total, rounds, round_len):
    _init(rank, world, port)
    p0, x, w, keys, inc = _run_restart_sharded(rank, world, B_total, rounds, round_len)
    np.savez(out + f".{rank}.npz", p0=p0, x=x, w=w, keys=np.array(keys), cnt=inc[0], gp=inc[1], a=inc[2])
    dist.destroy_process_group()


def test_restart_sharding_matches_single_process(tmp_path):
    """G = 2 ranks x 6 points reproduce G = 1 x 12 points exactly: per-point trajectories (Philox keyed by
    global point), the ERWA weights (global U_c), the any-solved / incumbent keys and the incumbent."""
    B_total, rounds, round_len = 12, 3, 4
    p0, x1, w1, keys1, inc1 = _run_restart_sharded(0, 1, B_total, rounds, round_len)
    out = str(tmp_path / "rs")
    mp.spawn(_restart_worker, args=(2, free_port(), out, B_total, rounds, round_len), nprocs=2, join=True)
    parts = [np.load(out + f".{r}.npz") for r in range(2)]
    x2 = np.concatenate([p["x"] for p in sorted(parts, key=lambda p: int(p["p0"]))])
    assert np.array_equal(x1, x2)
    for p in parts:
        assert np.array_equal(p["w"], w1)
        assert p["keys"].tolist() == keys1
        assert (int(p["cnt"]), int(p["gp"])) == (inc1[0], inc1[1])
        assert np.array_equal(p["a"], inc1[2])
    # the incumbent is a true minimiser of the falsified count over all global points
    Fo = OracleFormula.from_arrays(*synth.config1(4).arrays())
    cnt, _ = cdp.check(Fo, np.where(x1 < 0, -1.0, 1.0))
    assert inc1[0] == cnt.min() and inc1[1] == int(np.argmin(cnt))


def _solve_worker(rank, world, port, out, B_total):
    _init(rank, world, port)
    res = _solve(rank, world, B_total)
    np.savez(out + f".{rank}.npz", sat=res["sat"], a=res["assignment"], point=res["point"], rounds=res["rounds"],
             best=res["best_unsat"])
    dist.destroy_process_group()


def _planted():
    """planted 3-SAT n=40, m=176: the 16-point search needs 3 rounds and solves at global point 12 (rank 1 at G=2)"""
    z = np.random.default_rng(3).random(40) < 0.5
    return synth.random_ksat(40, 176, 3, 1, planted=z)


def _solve(rank, world, B_total, inst=None):
    inst = inst or _planted()
    Fo = OracleFormula.from_arrays(*inst.arrays())
    point0, B = D.point_range(B_total, world, rank)
    s = OracleSearch(Fo, B, 99, point0, osolve.Params(max_inner=2))

    def check(a):
        cnt, fw = cdp.check(Fo, np.where(np.asarray(a) < 0, -1.0, 1.0)[None])
        return int(cnt[0]), float(fw[0])
    return D.solve_sharded(s, check, round_len=2, max_rounds=40, rank=rank, world=world)


def test_solve_sharded_stops_all_ranks_with_the_same_verified_solution(tmp_path):
    """The restart-sharded solve loop: both ranks stop at the same round with the lowest solved global point's
    assignment, which the exact check verifies, and it is the single-process answer (G-independence)."""
    one = _solve(0, 1, 16)
    assert one["sat"] == 1 and one["rounds"] > 1 and one["point"] >= 8   # found by rank 1 after restarts
    out = str(tmp_path / "sv")
    mp.spawn(_solve_worker, args=(2, free_port(), out, 16), nprocs=2, join=True)
    parts = [np.load(out + f".{r}.npz") for r in range(2)]
    Fo = OracleFormula.from_arrays(*_planted().arrays())
    for p in parts:
        assert int(p["sat"]) == 1 and int(p["rounds"]) == one["rounds"] and int(p["point"]) == one["point"]
        assert np.array_equal(p["a"], one["assignment"])
        assert cdp.check(Fo, np.where(p["a"] < 0, -1.0, 1.0)[None])[0][0] == 0


def test_solve_sharded_unsat_returns_unknown_with_incumbent():
    """{x1, -x1} is unsatisfiable: UNKNOWN (never SAT), incumbent with one falsified clause."""
    Fo = OracleFormula.from_constraints(1, [(0, 0, 1.0, [1]), (0, 0, 1.0, [-1])])
    inst = synth.Instance("unsat", 1, Fo.kind, Fo.bound, Fo.weight, Fo.offsets, Fo.lits)
    s = OracleSearch(Fo, 4, 5, 0, osolve.Params(max_inner=5))

    def check(a):
        cnt, fw = cdp.check(Fo, np.where(np.asarray(a) < 0, -1.0, 1.0)[None])
        return int(cnt[0]), float(fw[0])
    r = D.solve_sharded(s, check, round_len=5, max_rounds=3)
    assert r["sat"] == 0 and r["best_unsat"] == 1 and r["rounds"] == 3
    assert inst.m == 2


# ---------------------------------------------------------------------------------------------- portfolio (f1)

STRATS = [osolve.Params(max_inner=2, policy="ROF", adaptive_weights=True),   # heuristics
          osolve.Params(max_inner=2, policy="R", adaptive_weights=False)]    # fresh random restarts, fixed weights


def _portfolio(rank, world, B=8):
    Fo = OracleFormula.from_arrays(*_planted().arrays())
    mine = D.portfolio_groups(world, 2, dist if world > 1 else None)[rank]
    searches = [(s, OracleSearch(Fo, B, 99, s * B, STRATS[s]), g) for s, g in mine]

    def check(a):
        cnt, fw = cdp.check(Fo, np.where(np.asarray(a) < 0, -1.0, 1.0)[None])
        return int(cnt[0]), float(fw[0])
    return D.solve_portfolio(searches, check, round_len=2, max_rounds=40, rank=rank, world=world)


def _portfolio_worker(rank, world, port, out):
    _init(rank, world, port)
    r = _portfolio(rank, world)
    np.savez(out + f".{rank}.npz", sat=r["sat"], a=r["assignment"], point=r["point"], rounds=r["rounds"],
             strategy=r["strategy"])
    dist.destroy_process_group()


def test_portfolio_groups_layout():
    assert D.portfolio_groups(1, 2) == [[(0, None), (1, None)]]
    lay = D.portfolio_groups(4, 2)
    assert [[s for s, _ in r] for r in lay] == [[0], [1], [0], [1]]


def test_portfolio_one_process_equals_one_strategy_per_rank(tmp_path):
    """f1 portfolio: both strategies on one process (one GPU, two searches) and one strategy per rank (two GPUs,
    "heuristics on / off per GPU group") stop at the same round with the same verified solution, because every point
    is keyed by its global index and each strategy's U_c stays within its group; the winner is at least as fast as
    either strategy alone."""
    one = _portfolio(0, 1)
    assert one["sat"] == 1
    out = str(tmp_path / "pf")
    mp.spawn(_portfolio_worker, args=(2, free_port(), out), nprocs=2, join=True)
    Fo = OracleFormula.from_arrays(*_planted().arrays())
    for r in range(2):
        p = np.load(out + f".{r}.npz")
        assert int(p["sat"]) == 1 and int(p["rounds"]) == one["rounds"] and int(p["point"]) == one["point"]
        assert int(p["strategy"]) == one["strategy"] and np.array_equal(p["a"], one["assignment"])
        assert cdp.check(Fo, np.where(p["a"] < 0, -1.0, 1.0)[None])[0][0] == 0
    for s in range(2):   # each strategy alone (same points, same keys) never beats the portfolio
        Fo2 = OracleFormula.from_arrays(*_planted().arrays())

        def check(a):
            cnt, fw = cdp.check(Fo2, np.where(np.asarray(a) < 0, -1.0, 1.0)[None])
            return int(cnt[0]), float(fw[0])
        alone = D.solve_portfolio([(s, OracleSearch(Fo2, 8, 99, s * 8, STRATS[s]), None)], check, round_len=2,
                                  max_rounds=40)
        assert (not alone["sat"]) or alone["rounds"] >= one["rounds"]
