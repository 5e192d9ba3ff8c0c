"""Multi-GPU orchestration of the hot path: one process per GPU,
torch.distributed for the process group (NCCL on GPUs, gloo in the CPU tests).

Restart sharding (configs c2 / c4).  The restart points of Alg. 1 are independent: rank r owns
the global points [r B, (r + 1) B) and a full replica of the formula.  Philox streams are keyed by the global
point index, so a point's trajectory does not depend on the number of GPUs.  The only exchanges are the
round-end collectives on library-owned device buffers:
  C2  U_c SUM   -- ERWA (Prop. 3) is defined over all p_t points on all GPUs;
  C1  any-solved: MIN of the library's solved key (lowest solved global point);
  C4  incumbent: MIN of the library's key (falsified count << 32 | global point), then a broadcast of its row.
C1 and C4 travel in one all-reduce of two int64 keys that ffsat_search_reduce writes on the device.

Constraint sharding (config c5, formulas too large for one GPU's throughput).  Each rank evaluates a
contiguous, cost-balanced range of the constraints for the full batch and the partial f, grad f and unsat
counts are summed with one all-reduce (C3).  f = sum_c w_c FE_c and grad f = sum over occurrences
(Def. 3 / Prop. 1) split exactly over any partition of the constraints.

Nothing here computes the method's arithmetic: every step runs in libffsat's kernels (or, in the CPU tests,
in whatever evaluator / search object the test passes in).
"""
from __future__ import annotations

import numpy as np

FAST_KINDS_MAX_K = 64   # OR / XOR / XNOR / NAE and the cardinality special cases take the product paths up to k = 64


def point_range(B_total: int, world: int, rank: int) -> tuple[int, int]:
    """(point0, B) of this rank: contiguous, sizes differing by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    base, extra = divmod(int(B_total), world)
    point0 = rank * base + min(rank, extra)
    return point0, base + (1 if rank < extra else 0)


def constraint_cost(kind, bound, offsets) -> np.ndarray:
    """Per-constraint work estimate: k for the one/two-product fast paths, 12 k M' instruction slots for the
    root-of-unity path (M' = floor((k + 1) / 2) roots)."""
    kind = np.asarray(kind)
    bound = np.asarray(bound)
    k = np.diff(np.asarray(offsets, np.int64))
    fast = (kind <= 2) | (kind == 5) | ((kind == 3) & ((bound <= 1) | (bound == k))) | \
           ((kind == 4) & ((bound == 0) | (bound >= k - 1)))
    fast &= k <= FAST_KINDS_MAX_K
    return np.where(fast, k, 12 * k * ((k + 1) // 2)).astype(np.float64)


def constraint_ranges(kind, bound, offsets, world: int) -> list[tuple[int, int]]:
    """Contiguous constraint ranges [c0, c1), one per rank, balanced by constraint_cost."""
    cost = constraint_cost(kind, bound, offsets)
    m = len(cost)
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")))
    cuts.append(m)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, m))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def sub_formula(n, kind, bound, weight, offsets, lits, c0: int, c1: int):
    """Arrays of constraints [c0, c1) over the same n variables."""
    offsets = np.asarray(offsets, np.int64)
    lo, hi = int(offsets[c0]), int(offsets[c1])
    return (int(n), np.asarray(kind)[c0:c1].copy(), np.asarray(bound)[c0:c1].copy(),
            np.asarray(weight)[c0:c1].copy(), offsets[c0:c1 + 1] - lo, np.asarray(lits)[lo:hi].copy())


class ShardedEval:
    """Constraint-sharded f / grad f / unsat: local partial evaluation of this rank's constraint range, then
    one SUM all-reduce of each output over the process group (C3).

    `evaluate(x) -> (f, grad, unsat)` evaluates this rank's sub-formula; by default a libffsat Context built
    from it (device tensors in, device tensors out).  Tests pass another evaluator."""

    def __init__(self, arrays, rank: int, world: int, group=None, evaluate=None, **ctx_kw):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank, self.world = rank, world
        n, kind, bound, weight, offsets, lits = arrays
        self.range = constraint_ranges(kind, bound, offsets, world)[rank]
        self.arrays = sub_formula(n, kind, bound, weight, offsets, lits, *self.range)
        self.ctx = None
        if evaluate is None:
            from .ffsat import Context
            self.ctx = Context.from_arrays(*self.arrays, **ctx_kw)

            def evaluate(x):
                return self.ctx.eval(x, grad=True, unsat=True)
        self._evaluate = evaluate

    def eval(self, x, chunks: int = 1):
        """chunks > 1 (and world > 1): the batch in `chunks` row blocks, the all-reduce of block i issued
        asynchronously so it overlaps the evaluation of block i + 1; the library's launch plan is
        batch-independent, so the results are the same bits as one block."""
        if self.world <= 1 or chunks <= 1 or x.shape[0] < 2 * chunks:
            f, g, u = self._evaluate(x)
            if self.world > 1:
                for t in (f, g, u):
                    self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
            return f, g, u
        import torch
        B = x.shape[0]
        cuts = [B * i // chunks for i in range(chunks + 1)]
        parts, works = [], []
        for i in range(chunks):
            fi, gi, ui = self._evaluate(x[cuts[i]:cuts[i + 1]])
            for t in (fi, gi, ui):
                works.append(self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group, async_op=True))
            parts.append((fi, gi, ui))
        for w in works:
            w.wait()
        return tuple(torch.cat([p[j] for p in parts]) for j in range(3))

    def eval_host(self, xh, fh, gh, uh=None, chunks: int = 1):
        """The same from pinned HOST buffers (x [B][n] in; f [B], grad [B][n], unsat [B] out, filled in place).  One
        rank: the library's host-buffer evaluation (ffsat_eval with host pointers: staged in chunks so the H2D copy of
        one overlaps the evaluation of another and the D2H copy of the previous one).  Several ranks: H2D, the
        sharded evaluation and its all-reduce, D2H."""
        import torch
        if self.world <= 1 and self.ctx is not None:
            from .ffsat import ffsat_eval
            ffsat_eval(self.ctx.ptr, xh, xh.shape[0], fh, gh, uh)
            return fh, gh, uh
        dev = torch.device("cuda", torch.cuda.current_device())
        f, g, u = self.eval(xh.to(dev, non_blocking=True), chunks=chunks)
        fh.copy_(f, non_blocking=True)
        gh.copy_(g, non_blocking=True)
        if uh is not None:
            uh.copy_(u, non_blocking=True)
        torch.cuda.synchronize()
        return fh, gh, uh


INT64_MAX = (1 << 63) - 1


class RestartSharded:
    """Alg. 1 over all ranks' points; this rank's B points start at global index point0 (the search was created with
    it, so its Philox streams and phase offsets are keyed by global point: trajectories do not depend on G).

    `search` is a libffsat Search (or a test double with the same methods): iterate(n), check(), reduce(),
    restart(U_global), begin_round(), tensors() -> {'x', 'unsat', 'U', 'keys', ...}, assignment(local_point).
    The any-solved flag and the incumbent are computed by the library (ffsat_search_reduce: device keys in global
    point indices); this class only moves them through the process group."""

    def __init__(self, search, round_len: int, rank: int = 0, world: int = 1, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.search, self.round_len = search, int(round_len)
        self.rank, self.world, self.group = rank, world, group
        self.T = search.tensors()
        self.point0 = int(getattr(search, "point0", 0))
        self.B = int(self.T["unsat"].numel())
        self.rounds = 0

    def _all_reduce(self, t, op):
        if self.world > 1:
            self.dist.all_reduce(t, op=op, group=self.group)

    def begin(self):
        self.search.begin_round()

    def exchange(self):
        """Round-end exchange without a host round trip: exact check of sgn(x) on every point (library; a point
        with no falsified constraint is marked solved and kept), C2 SUM of U_c over ranks (ERWA is defined over
        all p_t points), the library's any-solved / incumbent keys, then one MIN all-reduce of both keys
        (C1 + C4).  Returns the keys tensor [solved global point or INT64_MAX, (unsat << 32) | global point]."""
        s, T = self.search, self.T
        s.check()
        self._all_reduce(T["U"], self.dist.ReduceOp.SUM)
        s.reduce()
        self._all_reduce(T["keys"], self.dist.ReduceOp.MIN)
        return T["keys"]

    def restart(self):
        """ERWA with the global U_c and rephase (library), then the next round's start."""
        self.search.restart(self.T["U"])
        self.search.begin_round()
        self.rounds += 1

    def round_end(self):
        """exchange() + restart(), fully asynchronous (the timed bench step).  A solved point's assignment survives
        the rephase (the library keeps it), so the caller may poll the keys whenever it likes."""
        keys = self.exchange()
        self.restart()
        return keys

    def step(self, i: int):
        """One PGD iteration over the local batch; every round_len-th step also ends the round."""
        self.search.iterate(1)
        if (i + 1) % self.round_len == 0:
            return self.round_end()
        return None

    def fetch(self, global_point: int):
        """Assignment int8 [n] (-1 True / +1 False) of a global point, broadcast from the rank that owns it: the
        solved assignment if that point solved, else sgn of its current x (C4)."""
        torch = self.torch
        dev = self.T["unsat"].device
        lp = int(global_point) - self.point0
        mine = 0 <= lp < self.B
        n = self.T["x"].shape[1]
        a = torch.zeros(n, dtype=torch.int8, device=dev)
        if mine:
            a.copy_(torch.as_tensor(np.asarray(self.search.assignment(lp)), device=dev))
        if self.world > 1:
            owner = torch.tensor([self.rank if mine else -1], dtype=torch.int64, device=dev)
            self._all_reduce(owner, self.dist.ReduceOp.MAX)
            self.dist.broadcast(a, src=int(owner.item()), group=self.group)
        return a.cpu().numpy()

    def incumbent(self):
        """(falsified count, global point, assignment) of the best point over all ranks at a fresh check (C4): the
        library's incumbent key, MIN over ranks (lowest global index among equal counts: deterministic for any G),
        then the owner broadcasts its row."""
        keys = self.exchange()
        k = int(keys[1].item())
        cnt, gp = k >> 32, k & 0xFFFFFFFF
        return cnt, gp, self.fetch(gp)


def solve_sharded(search, check, round_len: int, max_rounds: int, rank: int = 0, world: int = 1, group=None,
                  timeout_s: float = 0.0, poll_every: int = 0):
    """Restart-sharded Alg. 1 over all ranks: every rank runs its points' PGD rounds; at each round end the
    ranks exchange U_c (C2) and the library's keys (C1 + C4).  All ranks stop together at the first poll whose
    any-solved key is set and return the solution of the lowest solved global point, verified by `check`
    (ffsat_check: the exact host count); otherwise they keep the best incumbent (fetched before the rephase) and
    return UNKNOWN after max_rounds or timeout_s (the same decision on every rank: rank 0's clock is broadcast).
    poll_every > 0 also polls the any-solved key every poll_every PGD iterations inside a round (trial points whose
    rounded assignment satisfied everything, captured by the library's PGD step).

    Returns dict(sat, assignment, best_unsat, point, rounds, iterations, seconds)."""
    import time
    import torch
    import torch.distributed as dist
    rs = RestartSharded(search, round_len, rank, world, group)
    keys_t = rs.T["keys"]
    t0 = time.perf_counter()
    best_cnt, best_gp, best_a = None, -1, None
    rs.begin()
    rounds = iters = 0
    stop = torch.zeros(1, dtype=torch.int32, device=rs.T["unsat"].device)
    poll = poll_every if 0 < poll_every < round_len else round_len

    def solved(gp):
        a = rs.fetch(gp)
        return a if check(a)[0] == 0 else None

    def out_of_time():
        if timeout_s <= 0:
            return False
        stop.fill_(1 if (rank == 0 and time.perf_counter() - t0 > timeout_s) else 0)
        if world > 1:
            dist.all_reduce(stop, op=dist.ReduceOp.MAX, group=group)
        return bool(int(stop.item()))

    def done(a, gp):
        return {"sat": 1, "assignment": a, "best_unsat": 0, "point": gp, "rounds": rounds, "iterations": iters,
                "seconds": time.perf_counter() - t0}

    for rounds in range(1, max_rounds + 1):
        it = 0
        while it + poll < round_len:                 # mid-round polls of the trial captures
            search.iterate(poll)
            it += poll
            iters += poll
            search.reduce()
            if world > 1:
                dist.all_reduce(keys_t, op=dist.ReduceOp.MIN, group=group)
            gp = int(keys_t[0].item())
            if gp != INT64_MAX:
                a = solved(gp)
                if a is not None:
                    return done(a, gp)
            if out_of_time():
                break
        else:
            search.iterate(round_len - it)
            iters += round_len - it
        keys = rs.exchange().cpu()                   # round end: exact check, U_c, keys
        solved_gp, inc = int(keys[0]), int(keys[1])
        if solved_gp != INT64_MAX:
            a = solved(solved_gp)
            if a is not None:
                return done(a, solved_gp)
        cnt, gp = inc >> 32, inc & 0xFFFFFFFF
        if best_cnt is None or cnt < best_cnt:
            best_a = rs.fetch(gp)
            best_cnt, best_gp = check(best_a)[0], gp
        if out_of_time():
            break
        rs.restart()
    return {"sat": 0, "assignment": best_a, "best_unsat": best_cnt, "point": best_gp, "rounds": rounds,
            "iterations": iters, "seconds": time.perf_counter() - t0}


def portfolio_groups(world: int, n_strategies: int, dist=None):
    """Strategy of each rank and the process groups of the portfolio ("employing multiple GPUs to
    simultaneously attempt different search strategies"): with world >= n_strategies, rank r runs strategy r mod n
    and strategy s's U_c are summed over the ranks running it (its own group); with fewer ranks than strategies
    every rank runs every strategy on a share of its points (groups None = the whole world).  Returns
    (strategies of this rank as a list of (strategy, group)) for every rank, in rank order."""
    if world >= n_strategies:
        groups = [None] * n_strategies
        if dist is not None and world > 1:
            # every rank must create every group, in the same order
            groups = [dist.new_group([r for r in range(world) if r % n_strategies == s]) for s in range(n_strategies)]
        return [[(r % n_strategies, groups[r % n_strategies])] for r in range(world)]
    return [[(s, None) for s in range(n_strategies)] for _ in range(world)]


def solve_portfolio(searches, check, round_len: int, max_rounds: int, rank: int = 0, world: int = 1, timeout_s: float = 0.0):
    """Portfolio of restart-sharded searches (Table 2 "Portfolio"): `searches` is
    this rank's list of (strategy, search, group) -- each search with its own strategy parameters (e.g. ERWA + (ROF) rephasing
    vs fixed weights + fresh random restarts) and point0 range disjoint from every other search of any rank (keys are
    global point indices); group is the process group over which that strategy's U_c are summed (None = this rank
    alone when world == 1, else the world).  Every round all searches run round_len PGD iterations, exchange U_c
    within their strategy, and the library's keys are MIN-reduced over this rank's searches and then over the world:
    the first solution of ANY strategy stops every rank (C1), verified by `check`.

    Returns dict(sat, assignment, best_unsat, point, strategy, rounds, seconds)."""
    import time
    import torch
    import torch.distributed as dist
    t0 = time.perf_counter()
    runs, strategies = [], []
    for strat, s, g in searches:
        T = s.tensors()
        runs.append((s, g, T, int(getattr(s, "point0", 0)), int(T["unsat"].numel())))
        strategies.append(int(strat))
        s.begin_round()
    dev = runs[0][2]["unsat"].device
    keys = torch.empty(2, dtype=torch.int64, device=dev)
    stop = torch.zeros(1, dtype=torch.int32, device=dev)
    best_cnt, best_gp, best_a = None, -1, None

    def owner_of(gp):
        for i, (s, g, T, p0, B) in enumerate(runs):
            if 0 <= gp - p0 < B:
                return i
        return -1

    def fetch(gp):
        i = owner_of(gp)
        n = runs[0][2]["x"].shape[1]
        a = torch.zeros(n, dtype=torch.int8, device=dev)
        if i >= 0:
            s, g, T, p0, B = runs[i]
            a.copy_(torch.as_tensor(np.asarray(s.assignment(gp - p0)), device=dev))
        if world > 1:
            owner = torch.tensor([rank if i >= 0 else -1], dtype=torch.int64, device=dev)
            dist.all_reduce(owner, op=dist.ReduceOp.MAX)
            dist.broadcast(a, src=int(owner.item()))
        return a.cpu().numpy()

    rounds = 0
    for rounds in range(1, max_rounds + 1):
        keys.fill_(INT64_MAX)
        for s, g, T, p0, B in runs:
            s.iterate(round_len)
            s.check()
            if world > 1:
                dist.all_reduce(T["U"], op=dist.ReduceOp.SUM, group=g)
            s.reduce()
            torch.minimum(keys, T["keys"], out=keys)
        if world > 1:
            dist.all_reduce(keys, op=dist.ReduceOp.MIN)
        k = keys.cpu()
        solved_gp, inc = int(k[0]), int(k[1])
        if solved_gp != INT64_MAX:
            a = fetch(solved_gp)
            if check(a)[0] == 0:
                i = owner_of(solved_gp)
                strat = torch.tensor([strategies[i] if i >= 0 else -1], dtype=torch.int64, device=dev)
                if world > 1:
                    dist.all_reduce(strat, op=dist.ReduceOp.MAX)
                return {"sat": 1, "assignment": a, "best_unsat": 0, "point": solved_gp, "strategy": int(strat.item()),
                        "rounds": rounds, "seconds": time.perf_counter() - t0}
        cnt, gp = inc >> 32, inc & 0xFFFFFFFF
        if best_cnt is None or cnt < best_cnt:
            best_a = fetch(gp)
            best_cnt, best_gp = check(best_a)[0], gp
        if timeout_s > 0:
            stop.fill_(1 if (rank == 0 and time.perf_counter() - t0 > timeout_s) else 0)
            if world > 1:
                dist.all_reduce(stop, op=dist.ReduceOp.MAX)
            if int(stop.item()):
                break
        for s, g, T, p0, B in runs:
            s.restart(T["U"])
            s.begin_round()
    return {"sat": 0, "assignment": best_a, "best_unsat": best_cnt, "point": best_gp, "strategy": -1, "rounds": rounds,
            "seconds": time.perf_counter() - t0}
