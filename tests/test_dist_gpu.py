"""Multi-rank paths of dist.py driving the REAL library (libffsat kernels) on one GPU: two ranks share cuda:0 over a
gloo process group (the box has one B200; NCCL refuses two ranks on one device, gloo moves the same device tensors).

  * ShardedEval (constraint sharding, C3): the all-reduced f / grad / unsat equal the oracle on the whole formula
    within the north_star tolerance, unsat exact.
  * RestartSharded (restart sharding, C1/C2/C4): 2 ranks x B/2 points reproduce the 1 x B run BIT FOR BIT after 3
    rounds -- points x, the search's ERWA weights, the per-round any-solved / incumbent keys and the incumbent --
    because the launch plan is batch-independent (ffsat_options.batch_ref) and every random draw is keyed by the
    global point (F7).
  * solve_sharded: both ranks stop at the same round with the same assignment, verified by the exact check.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import paper_2308_15020_b200 as P  # noqa: E402
from paper_2308_15020_b200 import dist as D  # noqa: E402
import synth  # noqa: E402
from oracle import cdp  # noqa: E402
from oracle.formula import OracleFormula  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)


# ------------------------------------------------------------------------------------------ constraint sharding

def _sharded_inst():
    return synth.random_mixed(n=120, m=700, seed=41, kmax=64)


def _sharded_worker(rank, world, port, out):
    _init(rank, world, port)
    inst = _sharded_inst()
    X = synth.points("U", 96, inst.n, 43)
    se = D.ShardedEval(inst.arrays(), rank, world, device=0, precision=32, batch_ref=96)
    f, g, u = se.eval(torch.from_numpy(X).cuda())
    # the overlapped C3 (two row blocks, the all-reduce of the first during the evaluation of the second)
    f2, g2, u2 = se.eval(torch.from_numpy(X).cuda(), chunks=2)
    torch.cuda.synchronize()
    same = bool(torch.equal(f, f2) and torch.equal(g, g2) and torch.equal(u, u2))
    np.savez(out + f".{rank}.npz", f=f.cpu().numpy(), g=g.cpu().numpy(), u=u.cpu().numpy(), r=np.array(se.range),
             same=same)
    dist.destroy_process_group()


def test_constraint_sharded_eval_real_library(tmp_path):
    out = str(tmp_path / "se")
    mp.spawn(_sharded_worker, args=(2, free_port(), out), nprocs=2, join=True)
    inst = _sharded_inst()
    X = synth.points("U", 96, inst.n, 43)
    Fo = OracleFormula.from_arrays(*inst.arrays())
    fo, go = cdp.evaluate(Fo, X.astype(np.float64))
    uo, _ = cdp.check(Fo, X.astype(np.float64))
    parts = [np.load(out + f".{r}.npz") for r in range(2)]
    assert 0 < int(parts[0]["r"][1]) < inst.m          # both ranks hold a proper share
    for p in parts:                                     # every rank holds the all-reduced result
        assert np.max(np.abs(p["f"] - fo) / np.maximum(1, np.abs(fo))) <= 1e-4
        assert np.max(np.abs(p["g"] - go) / np.maximum(1, np.abs(go))) <= 1e-4
        assert np.array_equal(p["u"], uo)
        assert bool(p["same"])                          # chunked / overlapped: the same bits


# ------------------------------------------------------------------------------------------ restart sharding

B_TOTAL, ROUNDS, ROUND_LEN, SEED = 256, 3, 6, 4242


def _restart_inst():
    return synth.config4_hybrid(2, n=300, m3=700, n_xor=60, kmax=24)


def _run_restart(rank, world):
    inst = _restart_inst()
    ctx = P.Context.from_instance(inst, device=0)
    point0, B = D.point_range(B_TOTAL, world, rank)
    s = ctx.search(B, seed=SEED, point0=point0, max_inner=ROUND_LEN)
    rs = D.RestartSharded(s, ROUND_LEN, rank, world)
    rs.begin()
    keys = []
    for i in range(ROUNDS * ROUND_LEN):
        k = rs.step(i)
        if k is not None:
            keys.append([int(v) for v in k.cpu()])
    s.iterate(2)                                       # a little into round 4: x mid-round, not just rephased
    T = s.tensors()
    x = T["x"].cpu().numpy().copy()
    w = T["weights"].cpu().numpy().copy()
    f = T["f"].cpu().numpy().copy()
    cnt, gp, a = rs.incumbent()
    return point0, x, w, f, keys, (cnt, gp, a)


def _restart_worker(rank, world, port, out):
    _init(rank, world, port)
    p0, x, w, f, keys, inc = _run_restart(rank, world)
    np.savez(out + f".{rank}.npz", p0=p0, x=x, w=w, f=f, keys=np.array(keys), cnt=inc[0], gp=inc[1], a=inc[2])
    dist.destroy_process_group()


def test_restart_sharded_two_ranks_bit_identical_to_one(tmp_path):
    torch.cuda.set_device(0)
    p0, x1, w1, f1, keys1, inc1 = _run_restart(0, 1)
    out = str(tmp_path / "rs")
    mp.spawn(_restart_worker, args=(2, free_port(), out), nprocs=2, join=True)
    parts = sorted([np.load(out + f".{r}.npz") for r in range(2)], key=lambda p: int(p["p0"]))
    assert np.array_equal(np.concatenate([p["x"] for p in parts]), x1)
    assert np.array_equal(np.concatenate([p["f"] for p in parts]), f1)
    for p in parts:
        assert np.array_equal(p["w"], w1)               # ERWA over the global U_c (C2), same on every rank
        assert p["keys"].tolist() == keys1              # C1 / C4 keys of every round
        assert (int(p["cnt"]), int(p["gp"])) == (inc1[0], inc1[1])
        assert np.array_equal(p["a"], inc1[2])
    # the incumbent is the exact minimiser over all global points of sgn(x) at that check
    inst = _restart_inst()
    Fo = OracleFormula.from_arrays(*inst.arrays())
    cnt, _ = cdp.check(Fo, np.where(x1 < 0, -1.0, 1.0))
    assert inc1[0] == cnt.min() and inc1[1] == int(np.argmin(cnt))


# ------------------------------------------------------------------------------------------ sharded solve

def _solve_inst():
    return synth.config4_hybrid(3, n=120, m3=430, n_xor=8, kmax=6)


def _solve(rank, world):
    inst = _solve_inst()
    ctx = P.Context.from_instance(inst, device=0)
    point0, B = D.point_range(128, world, rank)
    s = ctx.search(B, seed=7, point0=point0, max_inner=40)
    return D.solve_sharded(s, ctx.check, round_len=40, max_rounds=200, rank=rank, world=world)


def _solve_worker(rank, world, port, out):
    _init(rank, world, port)
    r = _solve(rank, world)
    np.savez(out + f".{rank}.npz", sat=r["sat"], a=r["assignment"], point=r["point"], rounds=r["rounds"])
    dist.destroy_process_group()


def test_solve_sharded_real_library(tmp_path):
    torch.cuda.set_device(0)
    one = _solve(0, 1)
    assert one["sat"] == 1
    out = str(tmp_path / "sv")
    mp.spawn(_solve_worker, args=(2, free_port(), out), nprocs=2, join=True)
    Fo = OracleFormula.from_arrays(*_solve_inst().arrays())
    for r in range(2):
        p = np.load(out + f".{r}.npz")
        assert int(p["sat"]) == 1 and int(p["rounds"]) == one["rounds"] and int(p["point"]) == one["point"]
        assert np.array_equal(p["a"], one["assignment"])
        assert cdp.check(Fo, np.where(p["a"] < 0, -1.0, 1.0)[None])[0][0] == 0


# ------------------------------------------------------------------------------------------ portfolio (f1)

PF_STRATS = [dict(policy="ROF", adaptive_weights=1), dict(policy="R", adaptive_weights=0)]


def _portfolio(rank, world):
    inst = _solve_inst()
    ctx = P.Context.from_instance(inst, device=0)
    mine = D.portfolio_groups(world, 2, dist if world > 1 else None)[rank]
    searches = [(s, ctx.search(64, seed=3, point0=64 * s, max_inner=30, **PF_STRATS[s]), g) for s, g in mine]
    return D.solve_portfolio(searches, ctx.check, round_len=30, max_rounds=200, rank=rank, world=world)


def _portfolio_worker(rank, world, port, out):
    _init(rank, world, port)
    r = _portfolio(rank, world)
    np.savez(out + f".{rank}.npz", sat=r["sat"], a=r["assignment"], point=r["point"], rounds=r["rounds"],
             strategy=r["strategy"])
    dist.destroy_process_group()


def test_portfolio_real_library(tmp_path):
    """Both strategies on one GPU (two searches) vs one strategy per rank: the same round, point, strategy and
    verified assignment."""
    torch.cuda.set_device(0)
    one = _portfolio(0, 1)
    assert one["sat"] == 1
    out = str(tmp_path / "pf")
    mp.spawn(_portfolio_worker, args=(2, free_port(), out), nprocs=2, join=True)
    for r in range(2):
        p = np.load(out + f".{r}.npz")
        assert int(p["sat"]) == 1 and int(p["rounds"]) == one["rounds"] and int(p["point"]) == one["point"]
        assert int(p["strategy"]) == one["strategy"] and np.array_equal(p["a"], one["assignment"])


# ------------------------------------------------------------------------------------------ NCCL on the library's buffers

def test_nccl_collectives_on_library_buffers():
    """The collectives dist.py issues, over an NCCL process group (one rank: the box has one GPU), on the library's own
    device buffers (zero-copy views of ffsat_search_get_buffers / the ShardedEval outputs): U_c SUM (int32), the keys
    MIN (int64), f / grad / unsat SUM (fp64 / fp32 / int32) and the assignment broadcast (int8) -- NCCL accepts
    every buffer and dtype, and a one-rank reduction leaves the values unchanged."""
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{free_port()}", rank=0, world_size=1)
    try:
        inst = _restart_inst()
        ctx = P.Context.from_instance(inst, device=0)
        s = ctx.search(64, seed=SEED, max_inner=ROUND_LEN)
        s.begin_round()
        s.iterate(3)
        s.check()
        s.reduce()
        T = s.tensors()
        torch.cuda.synchronize()
        U0, k0 = T["U"].clone(), T["keys"].clone()
        dist.all_reduce(T["U"], op=dist.ReduceOp.SUM)
        dist.all_reduce(T["keys"], op=dist.ReduceOp.MIN)
        a = torch.as_tensor(s.assignment(0), device="cuda")
        a0 = a.clone()
        dist.broadcast(a, src=0)
        torch.cuda.synchronize()
        assert torch.equal(T["U"], U0) and torch.equal(T["keys"], k0) and torch.equal(a, a0)
        se = D.ShardedEval(inst.arrays(), 0, 1, device=0, precision=32)
        X = torch.from_numpy(synth.points("U", 32, inst.n, 5)).cuda()
        f, g, u = se.eval(X)
        f0, g0, u0 = f.clone(), g.clone(), u.clone()
        for t in (f, g, u):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        torch.cuda.synchronize()
        assert torch.equal(f, f0) and torch.equal(g, g0) and torch.equal(u, u0)
    finally:
        dist.destroy_process_group()


def test_sharded_eval_host_buffers_one_rank():
    """ShardedEval.eval_host (pinned host buffers in and out; one rank: the library's pipelined host staging, here a
    c5-shaped 3-SAT formula on the grouped owner path in two 16-point chunks) gives the same bits as the device
    evaluation, and f / grad / unsat match the oracle."""
    torch.cuda.set_device(0)
    inst = synth.random_ksat(3001, 12600, 3, 41)
    se = D.ShardedEval(inst.arrays(), 0, 1, device=0, precision=32, path=2)
    X = synth.points("U", 32, inst.n, 42, np.float32)
    xh = torch.from_numpy(X).pin_memory()
    fh = torch.empty(32, dtype=torch.float64).pin_memory()
    gh = torch.empty((32, inst.n), dtype=torch.float32).pin_memory()
    uh = torch.empty(32, dtype=torch.int32).pin_memory()
    se.eval_host(xh, fh, gh, uh)
    f, g, u = se.eval(torch.from_numpy(X).cuda())
    assert torch.equal(fh, f.cpu()) and torch.equal(gh, g.cpu()) and torch.equal(uh, u.cpu())
    Fo = OracleFormula.from_arrays(*inst.arrays())
    fo, go = cdp.evaluate(Fo, X.astype(np.float64))
    assert np.max(np.abs(fh.numpy() - fo) / np.maximum(1, np.abs(fo))) <= 1e-4
    assert np.max(np.abs(gh.numpy() - go) / np.maximum(1, np.abs(go))) <= 1e-4
    assert np.array_equal(uh.numpy(), cdp.check(Fo, X.astype(np.float64))[0])
