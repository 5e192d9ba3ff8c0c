"""synth/ -- seeded synthetic instance and point generators shared by tests and bench.

Holds none of the method's arithmetic (no Walsh/Fourier coefficients, no products,
no gradients): only random structure, in the shapes PAPER.md's workloads and
BASELINE.json's configs name (recipes in DESIGN.md "Input recipe").  Both the
oracle and the CUDA path consume its output; neither is imported here.

Formula arrays: kind uint8 (0 OR, 1 XOR odd, 2 XNOR even, 3 CARD_GE, 4 CARD_LE, 5 NAE),
bound int32, weight float64, offsets int64[m+1], lits int32 (DIMACS, 1-based, sign = polarity).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

OR, XOR, XNOR, CARD_GE, CARD_LE, NAE = 0, 1, 2, 3, 4, 5
_TAG = {OR: "o", XOR: "x", XNOR: "xn", CARD_GE: "d", CARD_LE: "a", NAE: "n"}


@dataclass
class Instance:
    name: str
    n: int
    kind: np.ndarray
    bound: np.ndarray
    weight: np.ndarray
    offsets: np.ndarray
    lits: np.ndarray
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(len(self.kind))

    @property
    def n_lits(self) -> int:
        return int(self.offsets[-1])

    def arrays(self):
        return self.n, self.kind, self.bound, self.weight, self.offsets, self.lits

    def to_text(self, weighted: bool | None = None) -> str:
        """hnf / whnf text (SPEC S:102-103 grammar + `a`/`n` extension)."""
        if weighted is None:
            weighted = bool(np.any(self.weight != 1.0))
        out = [f"c {self.name}", f"p {'whnf' if weighted else 'hnf'} {self.n} {self.m}"]
        for c in range(self.m):
            ls = self.lits[self.offsets[c]:self.offsets[c + 1]]
            kd = int(self.kind[c])
            head = _TAG[kd] + (f" {int(self.bound[c])}" if kd in (CARD_GE, CARD_LE) else "")
            w = f"{float(self.weight[c])!r} " if weighted else ""
            out.append(f"{w}{head} " + " ".join(str(int(v)) for v in ls) + " 0")
        return "\n".join(out) + "\n"


def _build(name, n, cons_kind, cons_bound, cons_lits, weight=None, meta=None) -> Instance:
    m = len(cons_kind)
    lens = np.array([len(l) for l in cons_lits], dtype=np.int64)
    offsets = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    lits = np.concatenate([np.asarray(l, dtype=np.int32) for l in cons_lits]) if m else np.zeros(0, np.int32)
    return Instance(name, int(n), np.asarray(cons_kind, np.uint8), np.asarray(cons_bound, np.int32),
                    np.ones(m) if weight is None else np.asarray(weight, np.float64), offsets, lits, meta or {})


def _distinct_rows(rng, m, k, n):
    """m rows of k distinct variables in [0, n), uniformly (rejection of rows with repeats)."""
    V = rng.integers(0, n, size=(m, k))
    while True:
        S = np.sort(V, axis=1)
        bad = np.nonzero((S[:, 1:] == S[:, :-1]).any(axis=1))[0] if k > 1 else np.zeros(0, np.int64)
        if len(bad) == 0:
            return V
        V[bad] = rng.integers(0, n, size=(len(bad), k))


def random_ksat(n: int, m: int, k: int, seed: int, planted: np.ndarray | None = None, name=None) -> Instance:
    """Uniform random k-SAT, fixed clause length (k distinct vars, each negated w.p. 1/2).
    With `planted` (bool[n], True = variable True) clauses falsified by it are redrawn."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    V = _distinct_rows(rng, m, k, n)
    neg = rng.random((m, k)) < 0.5
    if planted is not None:
        while True:
            lit_true = planted[V] ^ neg
            bad = np.nonzero(~lit_true.any(axis=1))[0]
            if len(bad) == 0:
                break
            V[bad] = _distinct_rows(rng, len(bad), k, n)
            neg[bad] = rng.random((len(bad), k)) < 0.5
    lits = np.where(neg, -(V + 1), V + 1).astype(np.int32)
    offsets = np.arange(0, (m + 1) * k, k, dtype=np.int64)
    return Instance(name or f"rand{k}sat_n{n}_m{m}_s{seed}", n, np.zeros(m, np.uint8), np.zeros(m, np.int32),
                    np.ones(m), offsets, lits.reshape(-1), {"k": k, "planted": planted is not None})


# --- BASELINE.json configs -------------------------------------------------------------

def config1(seed: int = 0) -> Instance:
    """c1: random 3-SAT n=20, m=91 (SATLIB uf20-91 shape)."""
    return random_ksat(20, 91, 3, seed, name=f"c1_3sat_n20_m91_s{seed}")


def config2(seed: int = 0, planted: bool = False, alpha: float = 85.0) -> Instance:
    """c2: random 7-SAT n=200 at clause ratio alpha (85 default; 87.79 with planting)."""
    n = 200
    m = int(round(alpha * n))
    z = None
    if planted:
        z = np.random.default_rng(np.random.PCG64(seed + 7919)).random(n) < 0.5
    inst = random_ksat(n, m, 7, seed, planted=z, name=f"c2_7sat_n{n}_m{m}_s{seed}{'_planted' if planted else ''}")
    if z is not None:
        inst.meta["z"] = z
    return inst


def config3(seed: int = 0, n: int = 4096, m3: int = 8192, n_card: int = 32, kmin: int = 500, kmax: int = 2000) -> Instance:
    """c3: E2-shaped hybrid: planted 3-SAT plus CARD_LE(b) of length U{kmin..kmax},
    all-positive / all-negative w.p. 1/2, b = max(floor(k/2), T_z) so hidden z satisfies all."""
    rng = np.random.default_rng(np.random.PCG64(seed + 1000003))
    z = rng.random(n) < 0.5
    base = random_ksat(n, m3, 3, seed, planted=z)
    kinds = list(base.kind); bounds = list(base.bound)
    cl = [base.lits[base.offsets[c]:base.offsets[c + 1]] for c in range(base.m)]
    for _ in range(n_card):
        k = int(rng.integers(kmin, kmax + 1))
        vs = rng.choice(n, size=k, replace=False)
        negall = rng.random() < 0.5
        lits = -(vs + 1) if negall else vs + 1
        tz = int(np.sum(z[vs] ^ negall))
        kinds.append(CARD_LE); bounds.append(max(k // 2, tz)); cl.append(lits)
    return _build(f"c3_hybrid_card_n{n}_s{seed}", n, kinds, bounds, cl, meta={"z": z})


def config4_parity(seed: int = 0, N: int = 60, e: float = 0.25) -> Instance:
    """c4(i): parity learning with error: m = 2N XORs over uniform non-empty
    subsets, floor(e m) outputs flipped; success threshold ceil((1-e) m) satisfied."""
    rng = np.random.default_rng(np.random.PCG64(seed + 31337))
    z = rng.random(N) < 0.5
    m = 2 * N
    kinds, cl = [], []
    flips = set(rng.choice(m, size=int(np.floor(e * m)), replace=False).tolist())
    for i in range(m):
        while True:
            mask = rng.random(N) < 0.5
            if mask.any():
                break
        vs = np.nonzero(mask)[0]
        par = int(np.sum(z[vs])) & 1
        if i in flips:
            par ^= 1
        kinds.append(XOR if par else XNOR); cl.append(vs + 1)
    inst = _build(f"c4_parity_N{N}_s{seed}", N, kinds, [0] * m, cl,
                  meta={"z": z, "threshold": int(np.ceil((1 - e) * m))})
    return inst


def config4_hybrid(seed: int = 0, n: int = 1024, m3: int = 2048, n_xor: int = 512, kmin: int = 3, kmax: int = 64) -> Instance:
    """c4(ii): planted hybrid, 3-CNF plus XOR with k ~ U{kmin..kmax} consistent with hidden z."""
    rng = np.random.default_rng(np.random.PCG64(seed + 4242))
    z = rng.random(n) < 0.5
    base = random_ksat(n, m3, 3, seed, planted=z)
    kinds = list(base.kind); bounds = list(base.bound)
    cl = [base.lits[base.offsets[c]:base.offsets[c + 1]] for c in range(base.m)]
    for _ in range(n_xor):
        k = int(rng.integers(kmin, kmax + 1))
        vs = rng.choice(n, size=k, replace=False)
        neg = rng.random(k) < 0.5
        lits = np.where(neg, -(vs + 1), vs + 1)
        par = int(np.sum(z[vs] ^ neg)) & 1
        kinds.append(XOR if par else XNOR); bounds.append(0); cl.append(lits)
    return _build(f"c4_hybrid_n{n}_s{seed}", n, kinds, bounds, cl, meta={"z": z})


def config5(seed: int = 0, n: int = 1_000_000, m: int = 4_200_000) -> Instance:
    """c5: uniform random 3-SAT n=10^6, m=4.2*10^6 (ratio 4.2)."""
    return random_ksat(n, m, 3, seed, name=f"c5_3sat_n{n}_m{m}_s{seed}")


# --- PAPER.md App. D workloads --------------------------------------------------------

def rq1(name: str, seed: int = 0, n: int | None = None) -> Instance:
    """RQ1 gradient-timing formulas: xor1-3, card1-3, xor+card.
    Variables per formula are not stated in the paper; n defaults to 2x the longest constraint
    or 256, whichever is larger (DESIGN.md reading).  Cardinality bound = k/2 (at-least)."""
    spec = {"xor1": [(XOR, 200, 8)], "xor2": [(XOR, 400, 16)], "xor3": [(XOR, 800, 32)],
            "card1": [(CARD_GE, 50, 8)], "card2": [(CARD_GE, 100, 16)], "card3": [(CARD_GE, 200, 32)],
            "xor+card": [(XOR, 800, 8), (CARD_GE, 1, 32)]}[name]
    n = n or 256
    rng = np.random.default_rng(np.random.PCG64(seed + 99))
    kinds, bounds, cl = [], [], []
    for kd, cnt, k in spec:
        for _ in range(cnt):
            vs = rng.choice(n, size=k, replace=False)
            neg = rng.random(k) < 0.5
            kinds.append(kd); bounds.append(k // 2 if kd == CARD_GE else 0)
            cl.append(np.where(neg, -(vs + 1), vs + 1))
    return _build(f"rq1_{name}_s{seed}", n, kinds, bounds, cl)


def random_card(N: int, seed: int = 0) -> Instance:
    """Benchmark 1: m = 0.6N at-least-(l/2) constraints over l = 0.2N distinct
    variables, all positive or all negative w.p. 1/2."""
    rng = np.random.default_rng(np.random.PCG64(seed + 555))
    l, m = int(0.2 * N), int(0.6 * N)
    kinds, bounds, cl = [], [], []
    for _ in range(m):
        vs = rng.choice(N, size=l, replace=False)
        negall = rng.random() < 0.5
        kinds.append(CARD_GE); bounds.append(l // 2); cl.append(-(vs + 1) if negall else vs + 1)
    return _build(f"card_N{N}_s{seed}", N, kinds, bounds, cl)


def random_mixed(n: int, m: int, seed: int, kmax: int = 12) -> Instance:
    """Every kind, random lengths 1..kmax, random bounds and weights (parity-test coverage)."""
    rng = np.random.default_rng(np.random.PCG64(seed + 7))
    kinds, bounds, cl, w = [], [], [], []
    for _ in range(m):
        kd = int(rng.integers(0, 6))
        k = int(rng.integers(1, min(kmax, n) + 1))
        vs = rng.choice(n, size=k, replace=False)
        neg = rng.random(k) < 0.5
        b = int(rng.integers(0, k + 1)) if kd in (CARD_GE, CARD_LE) else 0
        kinds.append(kd); bounds.append(b); cl.append(np.where(neg, -(vs + 1), vs + 1))
        w.append(float(rng.choice([1.0, 0.5, 2.0, 0.25 + rng.random()])))
    return _build(f"mixed_n{n}_m{m}_s{seed}", n, kinds, bounds, cl, weight=w)


# --- points --------------------------------------------------------------------------------

def points(dist: str, B: int, n: int, seed: int, dtype=np.float32) -> np.ndarray:
    """[B][n] points: U uniform in [-1,1]; N near-corner (|x| = 1 - U(0,1e-3), random sign);
    C exact corners; Z mixed with exact zeros (tie rule) and +-1."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    if dist == "U":
        x = rng.uniform(-1.0, 1.0, size=(B, n))
    elif dist == "N":
        s = np.where(rng.random((B, n)) < 0.5, -1.0, 1.0)
        x = s * (1.0 - rng.uniform(0.0, 1e-3, size=(B, n)))
    elif dist == "C":
        x = np.where(rng.random((B, n)) < 0.5, -1.0, 1.0)
    elif dist == "Z":
        x = rng.choice(np.array([-1.0, -0.5, 0.0, -0.0, 0.5, 1.0]), size=(B, n))
    else:
        raise ValueError(dist)
    return np.ascontiguousarray(x.astype(dtype))


def planted_maxcut(l: int, k: int, seed: int = 0) -> Instance:
    """Benchmark 3: planted-partition graph of l clusters x k vertices; every unordered vertex pair
    is an edge with probability 1/2 (SPEC S:454 reading of the paper's size remark), weight 1 inside a cluster
    and 2 between clusters; one weighted XOR (odd) constraint per edge (u, v): satisfied iff u and v land on
    opposite sides, so the falsified weight is the uncut weight (Max-Cut as 2-XOR).
    meta: n, edges (u, v, w) arrays (0-based), cluster of each vertex."""
    rng = np.random.default_rng(np.random.PCG64(seed + 8080))
    n = l * k
    cluster = np.repeat(np.arange(l), k)
    iu, iv = np.triu_indices(n, 1)
    keep = rng.random(len(iu)) < 0.5
    u, v = iu[keep], iv[keep]
    w = np.where(cluster[u] == cluster[v], 1.0, 2.0)
    m = len(u)
    lits = np.stack([u + 1, v + 1], axis=1).astype(np.int32).reshape(-1)
    offsets = np.arange(0, 2 * m + 1, 2, dtype=np.int64)
    return Instance(f"maxcut_l{l}_k{k}_s{seed}", n, np.full(m, XOR, np.uint8), np.zeros(m, np.int32), w, offsets, lits,
                    {"edges_u": u, "edges_v": v, "edges_w": w, "cluster": cluster})
