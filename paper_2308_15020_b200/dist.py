"""Multi-GPU orchestration of the hot path: one process per GPU,
torch.distributed for the process group (NCCL on GPUs, gloo in the CPU tests).

Restart sharding (configs c2 / c4).  The restart points of Alg. 1 are independent: rank r owns
the global points [r B, (r + 1) B) and a full replica of the formula.  Philox streams are keyed by the global
point index, so a point's trajectory does not depend on the number of GPUs.  The only exchanges are the
round-end collectives on library-owned device buffers:
  C2  U_c SUM   -- ERWA (Prop. 3) is defined over all p_t points on all GPUs;
  C1  any-solved MAX;
  C4  incumbent: MIN over (falsified count, global point), then a broadcast of its assignment.

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

    def eval(self, x):
        f, g, u = self._evaluate(x)
        if self.world > 1:
            for t in (f, g, u):
                self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return f, g, u


class RestartSharded:
    """Alg. 1 over world x B points, this rank's B at global offset point0 (the search was created with it).

    `search` is a libffsat Search (or a test double with the same methods): iterate(n), check(),
    restart(U_global), begin_round(), tensors() -> {'x', 'unsat', 'U', ...}, assignment(local_point)."""

    def __init__(self, search, round_len: int, rank: int = 0, world: int = 1, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.search, self.round_len = search, int(round_len)
        self.rank, self.world, self.group = rank, world, group
        self.T = search.tensors()
        self.point0 = int(getattr(search, "point0", 0))
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.T["unsat"].device)
        self.rounds = 0

    def _all_reduce(self, t, op):
        if self.world > 1:
            self.dist.all_reduce(t, op=op, group=self.group)

    def begin(self):
        self.search.begin_round()

    def round_end(self):
        """Exact check of sgn(x) on every point, global U (C2) and any-solved flag (C1), ERWA + rephase with
        the global U, start of the next round.  Returns the any-solved flag tensor (not synchronised)."""
        s, T = self.search, self.T
        s.check()
        self._all_reduce(T["U"], self.dist.ReduceOp.SUM)
        self.flag.copy_((T["unsat"].min() == 0).to(self.flag.dtype).view(1))
        self._all_reduce(self.flag, self.dist.ReduceOp.MAX)
        s.restart(T["U"])
        s.begin_round()
        self.rounds += 1
        return self.flag

    def step(self, i: int):
        """One PGD iteration over the local batch; every round_len-th step also ends the round."""
        self.search.iterate(1)
        if (i + 1) % self.round_len == 0:
            return self.round_end()
        return None

    def incumbent(self):
        """(falsified count, global point, assignment int8 [n]) of the best current point over all ranks
        (C4): exact check of sgn(x) here, MIN over the packed key count << 32 | global point, then the
        owner broadcasts its row (lowest global index among equal counts: deterministic for any G)."""
        torch = self.torch
        self.search.check()
        unsat = self.T["unsat"]
        local = torch.argmin(unsat).item()  # lowest local index among the minima
        key = torch.tensor([(int(unsat[local].item()) << 32) | (self.point0 + local)], dtype=torch.int64,
                           device=unsat.device)
        self._all_reduce(key, self.dist.ReduceOp.MIN)
        k = int(key.item())
        cnt, gp = k >> 32, k & 0xFFFFFFFF
        B = unsat.numel()
        owner_local = gp - self.point0
        mine = 0 <= owner_local < B
        a = torch.zeros(self.T["x"].shape[1], dtype=torch.int8, device=unsat.device)
        if mine:
            a.copy_(torch.as_tensor(np.asarray(self.search.assignment(owner_local)), device=unsat.device))
        if self.world > 1:
            owner = torch.tensor([self.rank if mine else -1], dtype=torch.int64, device=unsat.device)
            self._all_reduce(owner, self.dist.ReduceOp.MAX)
            self.dist.broadcast(a, src=int(owner.item()), group=self.group)
        return cnt, gp, a.cpu().numpy()
