"""GPU parity: the CUDA path (through the C-ABI) against the oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): f and grad within 1e-4 * max(1, |ref|) elementwise on the
fp32 path, 1e-9 * max(1, |ref|) on the fp64 path; satisfied/unsat counts bit-exact.  The oracle
evaluates at exactly the values the GPU received (fp32 inputs promoted to fp64).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2308_15020_b200 as P
import synth
from conftest import golden
from oracle import cdp
from oracle import solve as osolve
from oracle.formula import OracleFormula, parse
from oracle.philox import uniform_pm1

TOL = {32: 1e-4, 64: 1e-9}


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def oracle_of(inst):
    return OracleFormula.from_arrays(*inst.arrays())


def compare(inst, X, precision=32, path=0, check_unsat=True, device_path=True, ctx=None):
    ctx = ctx or P.Context.from_instance(inst, precision=precision, path=path, device=0)
    dt = np.float64 if ctx.info["precision"] == 64 else np.float32
    X = np.ascontiguousarray(X, dtype=dt)
    if device_path:
        f, g, u = ctx.eval(torch.from_numpy(X).cuda(), grad=True, unsat=True)
        torch.cuda.synchronize()
        f, g, u = f.cpu().numpy(), g.cpu().numpy(), u.cpu().numpy()
    else:
        f, g, u = ctx.eval(X, grad=True, unsat=True)
    Fo = oracle_of(inst)
    fo, go = cdp.evaluate(Fo, X.astype(np.float64))
    tol = TOL[ctx.info["precision"]]
    ef = np.max(np.abs(f - fo) / np.maximum(1.0, np.abs(fo))) if len(fo) else 0.0
    eg = np.max(np.abs(g - go) / np.maximum(1.0, np.abs(go))) if g.size else 0.0
    assert ef <= tol, f"f rel err {ef:.3e} > {tol}"
    assert eg <= tol, f"grad rel err {eg:.3e} > {tol}"
    if check_unsat:
        uo, _ = cdp.check(Fo, X.astype(np.float64))
        assert np.array_equal(u, uo), "unsat counts differ"
    return ctx, ef, eg


# ------------------------------------------------------------------ eval parity, small sizes


@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("dist", ["U", "N", "C", "Z"])
def test_c1_3sat(path, dist):
    inst = synth.config1(0)
    for B in (1, 37):
        compare(inst, synth.points(dist, B, inst.n, 1000 + B), path=path)


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("path", [1, 2])
def test_mixed_all_kinds(precision, path):
    """Every kind, k = 1..64 (fast templated k <= 16, blocked 16 < k <= 64, root path for the
    cardinalities), random weights, ragged batch."""
    inst = synth.random_mixed(n=90, m=400, seed=11, kmax=64)
    compare(inst, synth.points("U", 77, inst.n, 3), precision=precision, path=path)
    compare(inst, synth.points("N", 33, inst.n, 4), precision=precision, path=path)


def test_host_buffers_equal_device_buffers():
    inst = synth.random_mixed(n=50, m=200, seed=12, kmax=30)
    X = synth.points("U", 40, inst.n, 5)
    ctx = P.Context.from_instance(inst, device=0)
    fh, gh, uh = ctx.eval(X, grad=True, unsat=True)
    fd, gd, ud = ctx.eval(torch.from_numpy(X).cuda(), grad=True, unsat=True)
    assert np.array_equal(fh, fd.cpu().numpy()) and np.array_equal(gh, gd.cpu().numpy())
    assert np.array_equal(uh, ud.cpu().numpy())


def test_deterministic_bitwise():
    inst = synth.config2(0)
    X = torch.from_numpy(synth.points("U", 256, inst.n, 7)).cuda()
    ctx = P.Context.from_instance(inst, device=0)
    a = ctx.eval(X)
    b = ctx.eval(X)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_tiled_and_global_paths_both_match_oracle():
    """The same formula forced onto the on-chip tiled path and onto the global path (different kernels, different
    partial sums: equal only within tolerance) -- each against the oracle."""
    inst = synth.random_mixed(n=60, m=300, seed=13, kmax=16)
    X = synth.points("U", 64, inst.n, 8)
    compare(inst, X, path=1)
    compare(inst, X, path=2)


@pytest.mark.parametrize("case", ["c2_wide", "mixed_tiled", "global_long", "root_fp64"])
def test_batch_independent_bits(case):
    """F7 / ffsat_options.batch_ref: a point's f, grad and unsat are the same BITS whatever batch it is evaluated in
    (whole batch, ragged sub-batches, single points, host buffers) -- the launch plan never sees the call's B."""
    if case == "c2_wide":
        inst = synth.config2(0)
    elif case == "mixed_tiled":
        inst = synth.random_mixed(n=90, m=400, seed=11, kmax=64)
    elif case == "global_long":
        inst = synth.config4_hybrid(0, n=1024, m3=1500, n_xor=200, kmax=64)
    else:
        inst = synth.config3(0, n=1500, m3=300, n_card=4, kmin=100, kmax=400)
    ctx = P.Context.from_instance(inst, device=0)
    X = synth.points("U", 200, inst.n, 55, ctx.dtype)
    xd = torch.from_numpy(X).cuda()
    f, g, u = ctx.eval(xd, grad=True, unsat=True)
    f, g, u = f.cpu().numpy(), g.cpu().numpy(), u.cpu().numpy()
    for lo, hi in ((0, 77), (77, 200), (5, 6), (199, 200)):
        fs, gs, us = ctx.eval(xd[lo:hi].contiguous(), grad=True, unsat=True)
        assert np.array_equal(fs.cpu().numpy(), f[lo:hi]) and np.array_equal(gs.cpu().numpy(), g[lo:hi])
        assert np.array_equal(us.cpu().numpy(), u[lo:hi])
    fh, gh, uh = ctx.eval(X, grad=True, unsat=True)
    assert np.array_equal(fh, f) and np.array_equal(gh, g) and np.array_equal(uh, u)
    fn, _, _ = ctx.eval(xd, grad=False)       # f without the gradient: the same fixed summation order
    assert np.array_equal(fn.cpu().numpy(), f)


@pytest.mark.parametrize("name", ["xor1", "xor2", "xor3", "card1", "card2", "card3", "xor+card"])
def test_rq1_workloads(name):
    """PAPER.md App. D RQ1 formulas: XOR k = 8..32 fast path, cardinality k = 8..32 root path."""
    inst = synth.rq1(name, seed=1)
    compare(inst, synth.points("U", 64, inst.n, 21))
    compare(inst, synth.points("N", 32, inst.n, 22))


@pytest.mark.parametrize("N", [20, 60])
def test_benchmark1_cardinality(N):
    inst = synth.random_card(N, seed=2)
    compare(inst, synth.points("U", 40, inst.n, 23))


def test_parity_learning_c4():
    inst = synth.config4_parity(0)
    compare(inst, synth.points("U", 50, inst.n, 24))
    compare(inst, synth.points("C", 50, inst.n, 25))


def test_c4_hybrid_small():
    inst = synth.config4_hybrid(0, n=300, m3=600, n_xor=120)
    compare(inst, synth.points("U", 64, inst.n, 26))


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("dist", ["U", "N", "Z"])
def test_long_fast_only_global(precision, dist):
    """Only 16 < k <= 64 fast constraints (XOR / XNOR / OR / NAE / AND kinds): the global path runs the long
    kernel alone (no short chunks); ragged batch spanning several point tiles."""
    rng = np.random.default_rng(31)
    n, kinds, bounds, cl = 200, [], [], []
    for j in range(90):
        k = int(rng.integers(17, 65))
        kd = [synth.OR, synth.XOR, synth.XNOR, synth.NAE, synth.CARD_GE][j % 5]
        vs = rng.choice(n, size=k, replace=False)
        neg = rng.random(k) < 0.5
        kinds.append(kd); bounds.append(k if kd == synth.CARD_GE else 0); cl.append(np.where(neg, -(vs + 1), vs + 1))
    inst = synth._build("long_fast", n, kinds, bounds, cl)
    ctx = P.Context.from_instance(inst, precision=precision, path=2, device=0)
    compare(inst, synth.points(dist, 70, inst.n, 29), precision=precision, ctx=ctx)


def test_long_kernel_64bit_gather_offsets():
    """the long-constraint kernel's x^T gather offset var * B * sizeof(T) exceeds 2^32 bytes when n B >= 2^30
    (fp32).  n = 1.1e6, B = 1024, XOR / OR constraints of length 17..64 over the highest variables (offsets up to
    4.5 GB): f, grad and unsat of sampled points against the oracle."""
    n, B = 1_100_000, 1024
    rng = np.random.default_rng(77)
    kinds, bounds, cl = [], [], []
    for j in range(120):
        k = int(rng.integers(17, 65))
        vs = n - 1 - rng.choice(60_000, size=k, replace=False)
        kinds.append([synth.XOR, synth.OR, synth.XNOR][j % 3]); bounds.append(0)
        cl.append(np.where(rng.random(k) < 0.5, -(vs + 1), vs + 1))
    inst = synth._build("long64", n, kinds, bounds, cl)
    ctx = P.Context.from_instance(inst, precision=32, device=0)
    assert ctx.info["path"] == 2
    g = torch.Generator(device="cuda").manual_seed(5)
    xd = torch.rand((B, n), generator=g, device="cuda", dtype=torch.float32) * 2 - 1
    f, gr, u = ctx.eval(xd, grad=True, unsat=True)
    idx = torch.tensor([0, 511, 1023], device="cuda")
    X = xd[idx].cpu().numpy().astype(np.float64)
    Fo = oracle_of(inst)
    fo, go = cdp.evaluate(Fo, X)
    uo, _ = cdp.check(Fo, X)
    assert np.max(np.abs(f[idx].cpu().numpy() - fo) / np.maximum(1, np.abs(fo))) <= 1e-4
    assert np.max(np.abs(gr[idx].cpu().numpy() - go) / np.maximum(1, np.abs(go))) <= 1e-4
    assert np.array_equal(u[idx].cpu().numpy(), uo)
    del xd, gr
    torch.cuda.empty_cache()


@pytest.mark.parametrize("precision", [32, 64])
def test_owner_computes_option(precision, monkeypatch):
    """FFSAT_OWN=1 (global path): constraints with k <= 3 take the owner-computes gradient (owner_grad_kernel: per
    variable, no T-buffer round trip), the rest the T buffer; f, grad, unsat against the oracle, mixed kinds incl.
    NAE (two product channels) and constant constraints, ragged batch; and bit-identical across batch splits."""
    monkeypatch.setenv("FFSAT_OWN", "1")
    inst = synth.random_mixed(n=90, m=400, seed=11, kmax=64)
    ctx = P.Context.from_instance(inst, precision=precision, path=2, device=0)
    assert ctx.info["n_own_lits"] > 0
    compare(inst, synth.points("U", 77, inst.n, 3), precision=precision, ctx=ctx)
    compare(inst, synth.points("Z", 40, inst.n, 4), precision=precision, ctx=ctx)
    X = torch.from_numpy(synth.points("U", 70, inst.n, 5, ctx.dtype)).cuda()
    f, g, u = ctx.eval(X, grad=True, unsat=True)
    f2, g2, u2 = ctx.eval(X[33:50].contiguous(), grad=True, unsat=True)
    assert torch.equal(f2, f[33:50]) and torch.equal(g2, g[33:50]) and torch.equal(u2, u[33:50])


@pytest.mark.parametrize("precision,ppt,lanes,k", [(32, 4, 8, 3), (32, 2, 8, 3), (32, 4, 4, 3), (32, 4, 2, 3),
                                                   (32, 2, 2, 3), (64, 2, 8, 3), (64, 2, 2, 3), (32, 4, 8, 2),
                                                   (64, 2, 4, 2), (32, 1, 1, 3), (64, 1, 1, 3), (32, 1, 1, 2)])
def test_owner_computes_sliced_uniform(precision, ppt, lanes, k, monkeypatch):
    """FFSAT_OWN=1 on a formula whose fast constraints are ALL short (uniform random k-SAT on the global path, n not a
    multiple of the block): x^T in lanes * ppt-point slices and the single-bucket grouped owner kernel
    (owner_grp_kernel, lanes threads per variable, ppt points per thread); f, grad, unsat against the oracle on a
    ragged batch (a partial last slice), and bit-identical when a point is evaluated in another batch / slice
    position."""
    monkeypatch.setenv("FFSAT_OWN", "1")
    monkeypatch.setenv("FFSAT_OWN_PPT", str(ppt))
    monkeypatch.setenv("FFSAT_OWN_LANES", str(lanes))
    inst = synth.random_ksat(3001, 12600, k, 5)
    ctx = P.Context.from_instance(inst, precision=precision, path=2, device=0)
    assert ctx.info["n_own_lits"] == ctx.info["n_lits"]
    compare(inst, synth.points("U", 21, inst.n, 6), precision=precision, ctx=ctx)
    compare(inst, synth.points("Z", 9, inst.n, 7), precision=precision, ctx=ctx)
    X = torch.from_numpy(synth.points("U", 37, inst.n, 8, ctx.dtype)).cuda()
    f, g, u = ctx.eval(X, grad=True, unsat=True)
    f2, g2, u2 = ctx.eval(X[5:30].contiguous(), grad=True, unsat=True)
    assert torch.equal(f2, f[5:30]) and torch.equal(g2, g[5:30]) and torch.equal(u2, u[5:30])


@pytest.mark.parametrize("precision", [32, 64])
def test_owner_grouped_default_on_single_short_bucket(precision, monkeypatch):
    """Default plan (no FFSAT_OWN): a global-path formula whose fast constraints are ONE bucket of 3-literal clauses
    takes the grouped owner kernel (owner_grp_kernel, 32-point slices in fp32, 16 in fp64); f, grad, unsat against
    the oracle over several slices with a ragged tail, and the same bits for a point in another batch position."""
    monkeypatch.delenv("FFSAT_OWN", raising=False)
    monkeypatch.delenv("FFSAT_OWN_PPT", raising=False)
    inst = synth.random_ksat(5003, 21000, 3, 9)
    ctx = P.Context.from_instance(inst, precision=precision, path=2, device=0)
    assert ctx.info["n_own_lits"] == ctx.info["n_lits"]
    compare(inst, synth.points("U", 70, inst.n, 10), precision=precision, ctx=ctx)
    compare(inst, synth.points("N", 33, inst.n, 11), precision=precision, ctx=ctx)
    compare(inst, synth.points("Z", 5, inst.n, 12), precision=precision, ctx=ctx)
    X = torch.from_numpy(synth.points("U", 70, inst.n, 13, ctx.dtype)).cuda()
    f, g, u = ctx.eval(X, grad=True, unsat=True)
    f2, g2, u2 = ctx.eval(X[31:69].contiguous(), grad=True, unsat=True)
    assert torch.equal(f2, f[31:69]) and torch.equal(g2, g[31:69]) and torch.equal(u2, u[31:69])


def test_owner_grouped_small_batches_and_host_chunks(monkeypatch):
    """Batches of <= 16 (<= 8) points take 2 (1) points per thread (16- / 8-point x^T slices) and host batches of
    9..32 points go as 8-point chunks: the same bits as the 4-per-thread evaluation of a larger batch (a point's
    arithmetic and summation order do not depend on the slice width), and the oracle on a 16-point batch."""
    monkeypatch.delenv("FFSAT_OWN", raising=False)
    monkeypatch.delenv("FFSAT_OWN_PPT", raising=False)
    inst = synth.random_ksat(4001, 16800, 3, 21)
    ctx = P.Context.from_instance(inst, precision=32, path=2, device=0)
    assert ctx.info["n_own_lits"] == ctx.info["n_lits"]
    compare(inst, synth.points("U", 16, inst.n, 22), ctx=ctx)
    X = synth.points("U", 70, inst.n, 23, ctx.dtype)
    xd = torch.from_numpy(X).cuda()
    f, g, u = ctx.eval(xd, grad=True, unsat=True)
    f, g, u = f.cpu().numpy(), g.cpu().numpy(), u.cpu().numpy()
    for lo, hi in ((0, 16), (16, 27), (40, 41), (50, 58)):
        fs, gs, us = ctx.eval(xd[lo:hi].contiguous(), grad=True, unsat=True)
        assert np.array_equal(fs.cpu().numpy(), f[lo:hi]) and np.array_equal(gs.cpu().numpy(), g[lo:hi])
        assert np.array_equal(us.cpu().numpy(), u[lo:hi])
    for lo, hi in ((0, 32), (10, 35), (3, 20)):   # host buffers: two 16-point chunks / one chunk
        fh, gh, uh = ctx.eval(np.ascontiguousarray(X[lo:hi]), grad=True, unsat=True)
        assert np.array_equal(fh, f[lo:hi]) and np.array_equal(gh, g[lo:hi]) and np.array_equal(uh, u[lo:hi])


@pytest.mark.parametrize("precision", [32, 64])
def test_owner_grouped_single_point_plan(precision, monkeypatch):
    """A single-point plan (batch_ref = 1: c5 at B = 1) takes the one-lane layout -- a warp over 32 variables, one
    point per thread, groups of 32 window-sorted variables; f, grad, unsat against the oracle at B = 1 and on a
    small batch (one pass per point), and the same bits for a point alone and inside the batch."""
    monkeypatch.delenv("FFSAT_OWN", raising=False)
    monkeypatch.delenv("FFSAT_OWN_LANES", raising=False)
    monkeypatch.delenv("FFSAT_OWN_PPT", raising=False)
    inst = synth.random_ksat(6007, 25200, 3, 31)
    ctx = P.Context.from_instance(inst, precision=precision, path=2, device=0, batch_ref=1)
    assert ctx.info["n_own_lits"] == ctx.info["n_lits"]
    compare(inst, synth.points("U", 1, inst.n, 32), precision=precision, ctx=ctx)
    compare(inst, synth.points("N", 1, inst.n, 33), precision=precision, ctx=ctx)
    compare(inst, synth.points("Z", 1, inst.n, 34), precision=precision, ctx=ctx)
    X = synth.points("U", 5, inst.n, 35, ctx.dtype)
    compare(inst, X, precision=precision, ctx=ctx)
    xd = torch.from_numpy(X).cuda()
    f, g, u = ctx.eval(xd, grad=True, unsat=True)
    f3, g3, u3 = ctx.eval(xd[3:4].contiguous(), grad=True, unsat=True)   # (a view 4-byte aligned only)
    assert torch.equal(f3, f[3:4]) and torch.equal(g3, g[3:4]) and torch.equal(u3, u[3:4])
    Z = torch.zeros((2, inst.n), dtype=xd.dtype, device="cuda")
    Z[1] = -0.0                                                            # signed zeros are canonicalised
    fz, gz, uz = ctx.eval(Z, grad=True, unsat=True)
    assert torch.equal(fz[0], fz[1]) and torch.equal(gz[0], gz[1]) and torch.equal(uz[0], uz[1])


def test_owner_grouped_with_root_path_slots(monkeypatch):
    """The grouped owner kernel also adds a variable's T slots (here the root-path terms of long at-most-b
    constraints sharing the variables with the 3-literal clauses), fp64, against the oracle."""
    monkeypatch.delenv("FFSAT_OWN", raising=False)
    inst = synth.config3(0, n=1500, m3=3000, n_card=3, kmin=100, kmax=300)
    ctx = P.Context.from_instance(inst, precision=64, path=2, device=0)
    assert 0 < ctx.info["n_own_lits"] < ctx.info["n_lits"]
    compare(inst, synth.points("U", 40, inst.n, 14), precision=64, ctx=ctx)
    compare(inst, synth.points("N", 9, inst.n, 15), precision=64, ctx=ctx)


def test_c4_hybrid_global_full_batch():
    """c4's shape (3-CNF + XOR k = 3..64, n = 1024) on the global path (short and long kernels) at B = 1024 (the
    bench launch configuration); oracle on every point of a 1024-point batch."""
    inst = synth.config4_hybrid(0)
    ctx = P.Context.from_instance(inst, precision=32, device=0)
    assert ctx.info["path"] == 2
    compare(inst, synth.points("U", 1024, inst.n, 30), ctx=ctx)


@pytest.mark.parametrize("k", [65, 130, 300, 700])
def test_long_cardinality_fp64(k):
    """Root path in fp64 at long k (group sizes 32..128), at-most-b, mixed with clauses."""
    inst = synth.config3(0, n=1500, m3=200, n_card=3, kmin=k, kmax=k)
    compare(inst, synth.points("U", 5, inst.n, 27))
    compare(inst, synth.points("N", 3, inst.n, 28))


@pytest.mark.parametrize("k", [256, 257, 300, 511, 512, 513, 1000, 2000, 2048, 2049])
def test_product_tree_path(k):
    """fp64 symmetric constraints of k >= 256 literals take the product-tree kernel (kernels_tree.cuh, ffsat_info
    n_tree_cons): f and the gradient against the T2 oracle at the fp64 tolerance on uniform, near-corner, corner and
    tie points, unsat exact; every kind of truth table (at-least-b, at-most-b with mixed signs, XOR / XNOR parity, OR,
    NAE), tree sizes around the powers of two (levels with and without a right child, partial leaf blocks)."""
    n = k + 40
    rng = np.random.default_rng(k)
    cons = []
    for kind, bnd in ((3, k // 3), (4, k // 2), (1, 0), (2, 0), (0, 0), (5, 0), (4, k - 1)):
        vs = rng.choice(n, size=k, replace=False) + 1
        lits = np.where(rng.random(k) < 0.5, -vs, vs).tolist()
        cons.append((kind, bnd, float(rng.uniform(0.5, 2.0)), lits))
    for _ in range(20):   # some short clauses on other paths alongside
        vs = rng.choice(n, size=3, replace=False) + 1
        cons.append((0, 0, 1.0, np.where(rng.random(3) < 0.5, -vs, vs).tolist()))
    Fo = OracleFormula.from_constraints(n, cons)
    inst = synth.Instance(f"tree{k}", n, Fo.kind, Fo.bound, Fo.weight, Fo.offsets, Fo.lits)
    ctx = P.Context.from_instance(inst, precision=64, device=0)
    # the tree must fit in one CTA's shared memory (k <= 2048); longer constraints stay on the root-of-unity path
    assert ctx.info["n_tree_cons"] == (7 if k <= 2048 else 0) and (ctx.info["tree_work"] > 0) == (k <= 2048)
    for B, dist in ((5, "U"), (3, "N"), (2, "C"), (3, "Z")):
        compare(inst, synth.points(dist, B, n, 300 + k + B), ctx=ctx)


def test_product_tree_matches_root_path(monkeypatch):
    """The same long constraints through the product tree and through the root-of-unity path (FFSAT_TREE=0): f and the
    gradient agree to 1e-12 (both fp64), unsat identical; and the tree path is deterministic bit for bit."""
    inst = synth.config3(0, n=3000, m3=300, n_card=6, kmin=400, kmax=1800)
    X = torch.from_numpy(synth.points("U", 8, inst.n, 41, np.float64)).cuda()
    ctx_t = P.Context.from_instance(inst, device=0)
    assert ctx_t.info["n_tree_cons"] == 6
    monkeypatch.setenv("FFSAT_TREE", "0")
    ctx_r = P.Context.from_instance(inst, device=0)
    assert ctx_r.info["n_tree_cons"] == 0
    ft, gt, ut = ctx_t.eval(X, unsat=True)
    fr, gr, ur = ctx_r.eval(X, unsat=True)
    ft2, gt2, _ = ctx_t.eval(X, unsat=True)
    torch.cuda.synchronize()
    assert torch.max(torch.abs(ft - fr) / torch.clamp(torch.abs(fr), min=1)).item() <= 1e-12
    assert torch.max(torch.abs(gt - gr) / torch.clamp(torch.abs(gr), min=1)).item() <= 1e-12
    assert torch.equal(ut, ur)
    assert torch.equal(ft, ft2) and torch.equal(gt, gt2)


def test_long_xor_or_root_path():
    """Fast kinds longer than 64 go to the root path (general truth table incl. parity)."""
    cons = [(1, 0, 1.0, list(range(1, 101))), (0, 0, 2.0, [-v for v in range(20, 120)]),
            (5, 0, 0.5, list(range(5, 90))), (2, 0, 1.0, list(range(3, 70)))]
    Fo = OracleFormula.from_constraints(130, cons)
    inst = synth.Instance("longfast", 130, Fo.kind, Fo.bound, Fo.weight, Fo.offsets, Fo.lits)
    compare(inst, synth.points("U", 9, 130, 29) * 0.3 + 0.5, precision=64)


def test_edge_cases():
    # single literal, single constraint, B = 1
    Fo = OracleFormula.from_constraints(1, [(0, 0, 1.0, [1])])
    inst = synth.Instance("unit", 1, Fo.kind, Fo.bound, Fo.weight, Fo.offsets, Fo.lits)
    compare(inst, np.array([[0.25]], np.float32))
    compare(inst, np.array([[0.0], [-0.0], [1.0], [-1.0]], np.float32))
    # constant constraints (GE b = 0, LE b = k) contribute -w and no gradient
    Fo = OracleFormula.from_constraints(3, [(3, 0, 1.0, [1, 2]), (4, 3, 2.0, [1, 2, 3]), (0, 0, 1.0, [2, -3])])
    inst = synth.Instance("const", 3, Fo.kind, Fo.bound, Fo.weight, Fo.offsets, Fo.lits)
    compare(inst, synth.points("U", 5, 3, 30))
    # empty batch
    ctx = P.Context.from_instance(synth.config1(0), device=0)
    f, g, u = ctx.eval(np.zeros((0, 20), np.float32), unsat=True)
    assert f.shape == (0,)
    # no constraints at all
    inst = synth.Instance("empty", 4, np.zeros(0, np.uint8), np.zeros(0, np.int32), np.zeros(0),
                          np.zeros(1, np.int64), np.zeros(0, np.int32))
    ctx = P.Context.from_instance(inst, device=0)
    f, g, u = ctx.eval(np.ones((3, 4), np.float32), unsat=True)
    assert np.all(f == 0) and np.all(g == 0) and np.all(u == 0)


def test_paper_examples_on_gpu():
    """Eg. 3: -59/128 and grad (19/64, 19/64, 33/64, 33/64); Eg. 8 weighted gradient."""
    for prec in (32, 64):
        ctx = P.Context.from_file(golden("eg2_eg3_card4_ge2.hnf"), precision=prec, device=0)
        f, g, _ = ctx.eval(np.array([[0.5, 0.5, -0.5, -0.5]], ctx.dtype))
        assert abs(f[0] + 59 / 128) < TOL[prec]
        assert np.max(np.abs(g[0] - np.array([19, 19, 33, 33]) / 64)) < TOL[prec]
    ctx = P.Context.from_file(golden("eg8_local.hnf"), device=0)
    ctx.set_weights(np.array([0.6, 1.0, 0.6]))
    _, g, _ = ctx.eval(np.array([[1, -1, -1, 1]], np.float32))
    assert np.max(np.abs(g[0] - np.array([-0.6, -0.4, -0.4, -0.6]))) < 1e-6
    assert np.allclose(ctx.get_weights(), [0.6, 1.0, 0.6])


# ------------------------------------------------------------------ full-size configs (sampled)


@pytest.mark.parametrize("dist", ["U", "N", "Z"])
def test_c2_full_size_sampled(dist):
    """c2 at full size (7-SAT n=200, m=17000, B=1024, the bench launch configuration) on uniform, near-corner (the
    late-PGD regime) and tie-heavy points; the oracle recomputes 12 sampled points at the full occurrence depth."""
    inst = synth.config2(0)
    X = synth.points(dist, 1024, inst.n, 1000)
    ctx = P.Context.from_instance(inst, device=0)
    f, g, u = ctx.eval(torch.from_numpy(X).cuda(), unsat=True)
    f, g, u = f.cpu().numpy(), g.cpu().numpy(), u.cpu().numpy()
    idx = np.array([0, 1, 31, 32, 33, 500, 511, 512, 767, 1000, 1022, 1023])
    Fo = oracle_of(inst)
    fo, go = cdp.evaluate(Fo, X[idx].astype(np.float64))
    uo, _ = cdp.check(Fo, X[idx].astype(np.float64))
    assert np.max(np.abs(f[idx] - fo) / np.maximum(1, np.abs(fo))) <= 1e-4
    assert np.max(np.abs(g[idx] - go) / np.maximum(1, np.abs(go))) <= 1e-4
    assert np.array_equal(u[idx], uo)


@pytest.mark.parametrize("B", [32, 256])
def test_c3_full_size_sampled(B):
    """c3 at full size (n=4096, 8192 clauses, 32 at-most-b of length 500..2000, fp64) at both bench batch sizes
    (B = 32: c3, B = 256: c3b256; the long constraints on the product tree), sampled points against the oracle."""
    inst = synth.config3(0)
    X = synth.points("U", B, inst.n, 1000, np.float64)
    ctx = P.Context.from_instance(inst, device=0)
    assert ctx.info["precision"] == 64
    f, g, u = ctx.eval(torch.from_numpy(X).cuda(), unsat=True)
    f, g, u = f.cpu().numpy(), g.cpu().numpy(), u.cpu().numpy()
    idx = np.array([0, 17, 31]) if B == 32 else np.array([0, 100, 199, 255])
    Fo = oracle_of(inst)
    fo, go = cdp.evaluate(Fo, X[idx])
    uo, _ = cdp.check(Fo, X[idx])
    assert np.max(np.abs(f[idx] - fo) / np.maximum(1, np.abs(fo))) <= 1e-9
    assert np.max(np.abs(g[idx] - go) / np.maximum(1, np.abs(go))) <= 1e-9
    assert np.array_equal(u[idx], uo)


def test_c5_full_size_sampled():
    """c5 at full size (3-SAT n=10^6, m=4.2*10^6, B=32, global path); oracle on 2 sampled points."""
    inst = synth.config5(0)
    X = synth.points("U", 32, inst.n, 1000)
    ctx = P.Context.from_instance(inst, device=0)
    assert ctx.info["path"] == 2
    f, g, u = ctx.eval(torch.from_numpy(X).cuda(), unsat=True)
    idx = np.array([0, 31])
    f, u = f.cpu().numpy()[idx], u.cpu().numpy()[idx]
    g = g[torch.from_numpy(idx).cuda()].cpu().numpy()
    Fo = oracle_of(inst)
    fo, go = cdp.evaluate(Fo, X[idx].astype(np.float64))
    uo, _ = cdp.check(Fo, X[idx].astype(np.float64))
    assert np.max(np.abs(f - fo) / np.maximum(1, np.abs(fo))) <= 1e-4
    assert np.max(np.abs(g - go) / np.maximum(1, np.abs(go))) <= 1e-4
    assert np.array_equal(u, uo)


# ------------------------------------------------------------------ solve-loop parity (per step)


def test_initial_points_and_rephase_match_oracle_philox():
    inst = synth.config1(0)
    ctx = P.Context.from_instance(inst, device=0)
    s = ctx.search(48, seed=77, point0=5)
    x0 = s.tensors()["x"].cpu().numpy().astype(np.float64)
    want = osolve.initial_points(77, range(5, 53), inst.n)
    assert np.array_equal(x0, want)
    s.begin_round()
    s.check()
    s.restart()
    torch.cuda.synchronize()
    x1 = s.tensors()["x"].cpu().numpy().astype(np.float64)
    want1 = osolve.rephase(x0, 77, 5, 1, osolve.Params())
    assert np.array_equal(x1, want1)
    # written out (reading #20): global b = 5 + i takes "ROF"[(0 + b) mod 3] at round 1
    for i in range(48):
        ph = "ROF"[(5 + i) % 3]
        want = x0[i] if ph == "O" else -x0[i] if ph == "F" else np.array(uniform_pm1(77, 5 + i, 1, inst.n))
        assert np.array_equal(x1[i], want)


EPS = {32: 2.0 ** -24, 64: 2.0 ** -53}


@pytest.mark.parametrize("precision", [32, 64])
def test_pgd_steps_match_oracle(precision):
    """Per-step parity of A8 ("same x and eta give the same x' and accept/reject"): before every
    iteration the oracle is re-synchronised to the GPU's state (x, eta, the search's weights); it recomputes f and
    grad at that x itself (T2 DP) and takes one Alg. 4 step; the GPU takes its step.  Then:
      * accept / reject agree bit-exactly wherever the oracle's Armijo margin exceeds what the evaluation tolerance
        can move (|margin| > 4 tol max(1, |f|)); eta follows exactly (halved / doubled, capped at eta0);
      * rejected points keep x bit-exactly; accepted points agree elementwise within the bound the arithmetic gives:
        x' = clip(x - eta g), so |x'_gpu - x'_or| <= eta |g_gpu - g_or| + rounding of the update
        <= eta tol max(1, |g_or|) + 2 eps (1 + eta |g_or|)  (eps = the dtype's unit roundoff);
      * the GPU's f at its new x matches the oracle's f there (eval parity)."""
    inst = synth.config1(3)
    ctx = P.Context.from_instance(inst, precision=precision, device=0)
    B = 64
    s = ctx.search(B, seed=9, max_inner=500, eta0=8.0)      # large steps: both accept and reject branches
    Fo = oracle_of(inst)
    Pp = osolve.Params(max_inner=500, eta0=8.0)
    tol, eps = TOL[precision], EPS[precision]
    s.begin_round()
    T = s.tensors()
    w = ctx.to_input_order(T["weights"].cpu().numpy().astype(np.float64))
    n_acc = n_rej = n_tie = 0
    for it in range(12):
        torch.cuda.synchronize()
        x = T["x"].cpu().numpy().astype(np.float64)
        eta = T["eta"].cpu().numpy().copy()
        st = osolve.State(x=x.copy(), f=None, g=None, eta=None, done=None, iters=None, w=w)
        osolve.start_round(Fo, st, Pp)
        st.eta = eta.copy()
        xp_or, fp_or, _, acc_or = osolve.pgd_iteration(Fo, st, Pp)
        s.iterate(1)
        torch.cuda.synchronize()
        x_new = T["x"].cpu().numpy().astype(np.float64)
        eta_new = T["eta"].cpu().numpy()
        f_new = T["f"].cpu().numpy()
        acc_gpu = eta_new == np.minimum(2 * eta, Pp.eta0)
        assert np.all(acc_gpu | (eta_new == 0.5 * eta)), "eta must be doubled (capped) or halved"
        f0, _ = cdp.evaluate_weighted(Fo, w, x)
        d = np.einsum("bn,bn->b", cdp.evaluate_weighted(Fo, w, x)[1], xp_or - x)
        margin = fp_or - (f0 + Pp.armijo_c1 * d)
        # a null step (the projection returns x itself, e.g. at a corner) is accepted by both sides exactly: f is
        # evaluated at the same bits (batch-independent plan) and f' <= f + 0 holds with equality
        null = np.all(xp_or == x, axis=1)
        assert np.all(acc_gpu[null]) and np.all(acc_or[null])
        clear = (np.abs(margin) > 4 * tol * np.maximum(1, np.abs(f0))) | null
        assert np.array_equal(acc_gpu[clear], acc_or[clear]), f"accept decisions differ at iteration {it}"
        n_tie += int((~clear).sum())
        rej = ~acc_gpu
        assert np.array_equal(x_new[rej], x[rej])
        _, g_or = cdp.evaluate_weighted(Fo, w, x)
        both = acc_gpu & acc_or
        bound = eta[:, None] * (tol * np.maximum(1, np.abs(g_or)) + 2 * eps * (1 + np.abs(g_or))) + 2 * eps
        assert np.all(np.abs(x_new - xp_or)[both] <= bound[both]), f"x' differs beyond the bound at iteration {it}"
        fo_new, _ = cdp.evaluate_weighted(Fo, w, x_new)
        assert np.max(np.abs(f_new - fo_new) / np.maximum(1, np.abs(fo_new))) <= tol
        n_acc += int(acc_gpu.sum())
        n_rej += int(rej.sum())
    assert n_acc > 0 and n_rej > 0, "the sequence must exercise both branches"
    assert n_tie <= 12 * B // 2, "most decisions must be clear of the tolerance band (the test has teeth)"


@pytest.mark.parametrize("precision", [32, 64])
def test_pgd_eta_schedule_hand_derived_on_gpu(precision):
    """The hand-derived Alg. 4 sequence of tests/test_oracle_pins.py::test_pgd_eta_schedule_hand_derived on the GPU
    (dyadic values: exact in fp32 and fp64): reject (eta 4 -> 2), reject (-> 1), accept at (-1/4, -1/4) (-> 2),
    accept at the stationary point (-> 4), then done at max_inner = 4."""
    cons = [(1, 0, 1.0, [1, 2]), (0, 0, 0.25, [1]), (0, 0, 0.25, [2])]
    Fo = OracleFormula.from_constraints(2, cons)
    ctx = P.Context.from_arrays(2, Fo.kind, Fo.bound, Fo.weight, Fo.offsets, Fo.lits, precision=precision, device=0)
    s = ctx.search(3, seed=1, eta0=4.0, max_inner=4)
    s.set_x(torch.zeros((3, 2), dtype=torch.float32 if precision == 32 else torch.float64, device="cuda"))
    s.begin_round()
    T = s.tensors()
    for eta_w, x_w, f_w in ((2.0, 0.0, 0.0), (1.0, 0.0, 0.0), (2.0, -0.25, -0.0625), (4.0, -0.25, -0.0625),
                            (4.0, -0.25, -0.0625)):
        s.iterate(1)
        torch.cuda.synchronize()
        assert np.all(T["eta"].cpu().numpy() == eta_w)
        assert np.all(T["x"].cpu().numpy() == x_w) and np.all(T["f"].cpu().numpy() == f_w)
    assert s.stats()["active"] == 0


@pytest.mark.parametrize("precision", [32, 64])
def test_fista_schedule_hand_derived_on_gpu(precision):
    """The hand-derived FISTA sequence of tests/test_oracle_pins.py::test_fista_schedule_hand_derived (reading #16b,
    P:939) on the GPU, dyadic values (exact in fp32 and fp64): from x = (0, 0), eta0 = 4 the first trial is (-1, -1);
    reject (eta 4 -> 2, trial (-1/2, -1/2)), reject (-> 1, trial (-1/4, -1/4)), accept with beta = 0 (-> 2, y = x+,
    next trial = y), accept with beta != 0 (-> 4, the next evaluation is y = x + beta (x - x_prev) = x, phase 0), then
    the y evaluation (phase 1 again)."""
    cons = [(1, 0, 1.0, [1, 2]), (0, 0, 0.25, [1]), (0, 0, 0.25, [2])]
    Fo = OracleFormula.from_constraints(2, cons)
    ctx = P.Context.from_arrays(2, Fo.kind, Fo.bound, Fo.weight, Fo.offsets, Fo.lits, precision=precision, device=0)
    s = ctx.search(3, seed=1, eta0=4.0, max_inner=50, accel=1, adaptive_weights=0)
    s.set_x(torch.zeros((3, 2), dtype=torch.float32 if precision == 32 else torch.float64, device="cuda"))
    s.begin_round()
    T = s.tensors()
    torch.cuda.synchronize()
    assert np.all(T["xp"].cpu().numpy() == -1.0) and np.all(T["phase"].cpu().numpy() == 1)
    want = [(2.0, -0.5, 1, 0.0), (1.0, -0.25, 1, 0.0), (2.0, -0.25, 1, -0.25), (4.0, -0.25, 0, -0.25),
            (4.0, -0.25, 1, -0.25)]
    for k, (eta_w, xp_w, ph_w, x_w) in enumerate(want):
        s.iterate(1)
        torch.cuda.synchronize()
        assert np.all(T["eta"].cpu().numpy() == eta_w), k
        assert np.all(T["xp"].cpu().numpy() == xp_w), k
        assert np.all(T["phase"].cpu().numpy() == ph_w), k
        assert np.all(T["x"].cpu().numpy() == x_w), k
    assert np.all(T["f"].cpu().numpy() == -0.0625) and np.all(T["f_y"].cpu().numpy() == -0.0625)
    t2 = (1 + np.sqrt(1 + 4 * ((1 + 5 ** 0.5) / 2) ** 2)) / 2
    assert np.all(np.abs(T["t"].cpu().numpy() - t2) < 1e-15)
    assert np.all(T["grad"].cpu().numpy() == 0.0)   # the gradient at y = the stationary point (Eg. 7)


@pytest.mark.parametrize("precision,path", [(32, 0), (32, 4), (64, 0)])
def test_fista_steps_match_oracle(precision, path):
    """Per-step parity of the FISTA mode (reading #16b) against oracle/solve.py:fista_iteration: before every iteration
    the oracle is re-synchronised to the GPU's state (x, x_prev, y, the point to evaluate, t, eta, phase) and evaluates
    f, grad at y and at that point itself (T2 DP); both take one step.  Then:
      * the action (y consumed / accept / reject) agrees wherever the oracle's margin against the quadratic upper
        bound exceeds what the evaluation tolerance can move, eta and t follow exactly;
      * accepted points: x is the evaluated point bit-exactly and x_prev the old x; the next point agrees within the
        update's bound -- a projected trial clip(y - eta g_y): eta tol max(1, |g|) + rounding; an extrapolation
        x + beta (x - x_prev): rounding only;
      * rejected points keep x bit-exactly.
    path 0 in fp32 is the TMEM kernel with the reduction fused into the FISTA step; path 4 the shared-memory tiled
    kernel with the separate step; fp64 the general path."""
    inst = synth.config1(3)
    ctx = P.Context.from_instance(inst, precision=precision, device=0, path=path)
    if precision == 32:
        assert ctx.info["wide"] == (2 if path == 0 else 1)
    B = 64
    s = ctx.search(B, seed=9, max_inner=500, eta0=8.0, accel=1)
    Fo = oracle_of(inst)
    Pp = osolve.Params(max_inner=500, eta0=8.0)
    tol, eps = TOL[precision], EPS[precision]
    s.begin_round()
    T = s.tensors()
    w = ctx.to_input_order(T["weights"].cpu().numpy().astype(np.float64))
    seen = {"y": 0, "accept": 0, "reject": 0}
    n_tie = 0
    get = lambda k: T[k].cpu().numpy().astype(np.float64)
    for it in range(16):
        torch.cuda.synchronize()
        x, xm, y, xp = get("x"), get("x_prev"), get("y"), get("xp")
        t, eta, phase = get("t"), get("eta"), T["phase"].cpu().numpy().copy()
        fy_o, gy_o = cdp.evaluate_weighted(Fo, w, y)
        f_o, g_o = cdp.evaluate_weighted(Fo, w, x)
        st = osolve.FistaState(x=x.copy(), f=f_o, g=g_o, xm=xm.copy(), y=y.copy(), fy=fy_o, gy=gy_o, xp=xp.copy(),
                               t=t.copy(), eta=eta.copy(), phase=phase.astype(np.int64), done=np.zeros(B, bool),
                               iters=np.zeros(B, np.int64), w=w)
        fp_o, gp_o = cdp.evaluate_weighted(Fo, w, xp)
        acts = osolve.fista_iteration(Fo, st, Pp)
        s.iterate(1)
        torch.cuda.synchronize()
        x2, xm2, xp2 = get("x"), get("x_prev"), get("xp")
        eta2, t2 = get("eta"), get("t")
        dx = xp - y
        margin = fp_o - (fy_o + np.einsum("bn,bn->b", gy_o, dx) + np.einsum("bn,bn->b", dx, dx) / (2 * eta))
        for b in range(B):
            if phase[b] == 0:
                act = "y"
                assert eta2[b] == eta[b] and t2[b] == t[b]
            elif eta2[b] == min(2 * eta[b], Pp.eta0) and t2[b] != t[b]:
                act = "accept"
            else:
                act = "reject"
                assert eta2[b] == 0.5 * eta[b] and t2[b] == t[b]
            clear = phase[b] == 0 or abs(margin[b]) > 4 * tol * max(1.0, abs(fy_o[b]))
            if not clear:
                n_tie += 1
                continue
            assert act == acts[b], f"iteration {it} point {b}: GPU {act}, oracle {acts[b]}"
            seen[act] += 1
            assert eta2[b] == st.eta[b] and t2[b] == st.t[b]
            if act == "accept":
                assert np.array_equal(x2[b], xp[b]) and np.array_equal(xm2[b], x[b])
                if st.phase[b] == 0:   # extrapolation point: rounding of x + beta (x - x_prev) only
                    assert np.all(np.abs(xp2[b] - st.xp[b]) <= 8 * eps * (1 + np.abs(st.xp[b])))
                    continue
            else:
                assert np.array_equal(x2[b], x[b])
            # a new trial clip(y - eta g_y): y is the evaluated point after consuming y or a beta = 0 accept (its
            # gradient comes from this evaluation), the old y after a reject; the GPU's g_y differs from the
            # oracle's within the evaluation tolerance
            g_new = gy_o[b] if act == "reject" else gp_o[b]
            gmax = max(1.0, float(np.max(np.abs(g_new))))
            trial_bound = st.eta[b] * (tol * gmax + 2 * eps * (1 + gmax)) + 2 * eps
            assert np.all(np.abs(xp2[b] - st.xp[b]) <= trial_bound), f"trial differs at iteration {it} point {b}"
    assert all(v > 0 for v in seen.values()), seen
    assert n_tie <= 16 * B // 4, "most decisions must be clear of the tolerance band (the test has teeth)"


def test_fista_solve_small_formulas():
    """ffsat_solve with accel = 1: the Eg. 7 formula and uniform random 3-SAT (c1) solve, every SAT answer verified by
    the exact check and the oracle; the UNSAT pair {x1, -x1} stays UNKNOWN."""
    ctx = P.Context.from_file(golden("eg7_saddle.hnf"), device=0)
    r, a = ctx.solve(batch=8, max_restarts=5, seed=1, max_inner=50, accel=1)
    assert r["sat"] == 1 and ctx.check(a)[0] == 0
    Fo = OracleFormula.from_constraints(1, [(0, 0, 1.0, [1]), (0, 0, 1.0, [-1])])
    ctx = P.Context.from_arrays(1, Fo.kind, Fo.bound, Fo.weight, Fo.offsets, Fo.lits, device=0)
    r, a = ctx.solve(batch=8, max_restarts=3, seed=1, max_inner=30, accel=1)
    assert r["sat"] == 0 and r["best_unsat"] == 1
    solved = 0
    for seed in range(3):
        inst = synth.config1(seed)
        ctx = P.Context.from_instance(inst, device=0)
        r, a = ctx.solve(batch=256, max_restarts=20, seed=seed, max_inner=100, accel=1)
        if r["sat"]:
            solved += 1
            assert ctx.check(a)[0] == 0
            assert cdp.check(oracle_of(inst), np.where(a < 0, -1.0, 1.0)[None])[0][0] == 0
    assert solved >= 1


def test_check_U_and_erwa_match_oracle():
    """Round-end check (A9) and ERWA (A10): unsat[b] exact; U_c exact PER CONSTRAINT (the device array is in
    position order, mapped back with Context.order()); the search's weights after the restart equal Prop. 3's
    update of the oracle within the fp32 rounding of the weight store; the context's own weights are untouched."""
    inst = synth.config2(1)
    ctx = P.Context.from_instance(inst, device=0)
    s = ctx.search(64, seed=3)
    s.check()
    torch.cuda.synchronize()
    T = s.tensors()
    x = T["x"].cpu().numpy().astype(np.float64)
    Fo = oracle_of(inst)
    cnt, _, U = cdp.check(Fo, x, want_U=True)
    assert np.array_equal(T["unsat"].cpu().numpy(), cnt)
    assert np.array_equal(ctx.to_input_order(T["U"].cpu().numpy()), U)
    s.restart()
    torch.cuda.synchronize()
    w_dev = ctx.to_input_order(T["weights"].cpu().numpy().astype(np.float64))
    w_or = osolve.erwa_update(np.ones(Fo.m), U, 0.4)
    assert np.max(np.abs(w_dev - w_or)) <= 2.0 ** -24
    assert np.array_equal(ctx.get_weights(), np.ones(Fo.m))


def test_round_end_check_marks_solved_and_keys():
    """A point whose sgn(x) satisfies everything at the round-end check is marked solved and its assignment kept
    through the rephase; ffsat_search_reduce's keys are the lowest solved global point and the exact
    (falsified count, global point) minimum."""
    inst = synth.config2(0, planted=True, alpha=40.0)
    z = inst.meta["z"]
    ctx = P.Context.from_instance(inst, device=0)
    B, point0 = 40, 1000
    s = ctx.search(B, seed=12, point0=point0)
    X = synth.points("U", B, inst.n, 71)
    X[13] = np.where(z, -0.5, 0.5)          # the planted assignment (True = negative coordinate)
    X[29] = np.where(z, -0.25, 0.75)
    s.set_x(torch.from_numpy(X).cuda())
    s.check()
    s.reduce()
    torch.cuda.synchronize()
    T = s.tensors()
    Fo = oracle_of(inst)
    cnt, _ = cdp.check(Fo, X.astype(np.float64))
    keys = T["keys"].cpu().numpy()
    assert keys[0] == point0 + 13
    i = int(np.argmin(cnt))
    assert keys[1] == (int(cnt[i]) << 32) | (point0 + i)
    s.restart()
    torch.cuda.synchronize()
    a = s.assignment(13)
    assert np.array_equal(a, np.where(z, -1, 1)) and ctx.check(a)[0] == 0
    st = s.stats()
    assert st["solved_point"] == point0 + 13


def test_solve_small_formulas():
    ctx = P.Context.from_file(golden("eg7_saddle.hnf"), device=0)
    r, a = ctx.solve(batch=8, max_restarts=5, seed=1, max_inner=50)
    assert r["sat"] == 1 and ctx.check(a)[0] == 0
    Fo = OracleFormula.from_constraints(1, [(0, 0, 1.0, [1]), (0, 0, 1.0, [-1])])
    ctx = P.Context.from_arrays(1, Fo.kind, Fo.bound, Fo.weight, Fo.offsets, Fo.lits, device=0)
    r, a = ctx.solve(batch=8, max_restarts=3, seed=1, max_inner=30)
    assert r["sat"] == 0 and r["best_unsat"] == 1
    for seed in range(3):
        inst = synth.config1(seed)
        ctx = P.Context.from_instance(inst, device=0)
        r, a = ctx.solve(batch=256, max_restarts=20, seed=seed, max_inner=100)
        if r["sat"]:
            assert ctx.check(a)[0] == 0
            assert cdp.check(oracle_of(inst), np.where(a < 0, -1.0, 1.0)[None])[0][0] == 0


def test_solve_planted_hybrid():
    inst = synth.config4_hybrid(1, n=200, m3=400, n_xor=20, kmax=8)
    ctx = P.Context.from_instance(inst, device=0)
    r, a = ctx.solve(batch=512, max_restarts=30, seed=2, max_inner=200)
    if r["sat"]:
        assert ctx.check(a)[0] == 0
    assert r["best_unsat"] >= 0


# ------------------------------------------------------------------ kernel variants and launch geometries


@pytest.mark.parametrize("k,kind,bnd", [(3, 0, 0), (7, 0, 0), (5, 1, 0), (16, 2, 0), (4, 3, 4), (6, 4, 0), (5, 4, 4)])
def test_wide_and_narrow_tiled_kernels(k, kind, bnd):
    """Uniform single-channel formulas take the 64-point (two points per lane, f32x2) tiled kernel; path 3
    forces the 32-point kernel.  Both against the oracle, odd and single-point batches, n at the wide limit.
    Kinds cover every truth-bit reduction of the wide kernel: OR, XOR, XNOR, AND (at least k), NOR (at most
    0), NAND (at most k - 1)."""
    n = 430
    rng = np.random.default_rng(5)
    m = 3 * n
    lits = []
    for _ in range(m):
        vs = rng.choice(n, size=k, replace=False) + 1
        lits.append(np.where(rng.random(k) < 0.5, -vs, vs))
    inst = synth._build(f"uniform_k{k}_kind{kind}", n, [kind] * m, [bnd] * m, lits)
    for path, wide in ((0, 1), (3, 0)):
        ctx = P.Context.from_instance(inst, precision=32, path=path, device=0)
        assert ctx.info["path"] == 1 and ctx.info["wide"] == wide
        for B, dist in ((65, "U"), (1, "N"), (128, "Z")):
            compare(inst, synth.points(dist, B, n, 100 + B), ctx=ctx)


@pytest.mark.parametrize("k,kind,bnd", [(3, 0, 0), (7, 0, 0), (5, 1, 0), (16, 2, 0), (4, 3, 4), (6, 4, 0), (5, 4, 4), (1, 0, 0)])
def test_tmem_tiled_kernel(k, kind, bnd):
    """n <= 256: the 64-point kernel keeps its gradient tile in tensor memory (ffsat_info wide == 2; four warp-group
    partial tiles in the TMEM lane quadrants).  Against the oracle for every truth-bit reduction, on ragged and single-point
    batches and n at the TMEM limit, with and without the fused check (f-only evaluations skip it); path 4 forces the
    shared-memory 64-point kernel on the same formula, also against the oracle."""
    n = 256 if k != 16 else 200
    rng = np.random.default_rng(k * 10 + kind)
    m = 40 * n // k
    lits = []
    for _ in range(m):
        vs = rng.choice(n, size=k, replace=False) + 1
        lits.append(np.where(rng.random(k) < 0.5, -vs, vs))
    inst = synth._build(f"tmem_k{k}_kind{kind}", n, [kind] * m, [bnd] * m, lits)
    for path, wide in ((0, 2), (4, 1)):
        ctx = P.Context.from_instance(inst, precision=32, path=path, device=0)
        assert ctx.info["path"] == 1 and ctx.info["wide"] == wide
        for B, dist in ((130, "U"), (1, "N"), (64, "Z"), (300, "N")):
            compare(inst, synth.points(dist, B, n, 200 + B), ctx=ctx)
        X = synth.points("U", 97, n, 17)
        f, _, _ = ctx.eval(torch.from_numpy(X).cuda(), grad=False)
        fo, _ = cdp.evaluate(oracle_of(inst), X.astype(np.float64))
        assert np.max(np.abs(f.cpu().numpy() - fo) / np.maximum(1, np.abs(fo))) <= 1e-4


def test_uniform_check_mixed_rules():
    """The uniform-k sgn check with different rules per constraint (OR / XOR / XNOR / NAE, k = 5)."""
    n, m, k = 120, 700, 5
    rng = np.random.default_rng(9)
    kinds = rng.choice([0, 1, 2, 5], size=m)
    lits = []
    for _ in range(m):
        vs = rng.choice(n, size=k, replace=False) + 1
        lits.append(np.where(rng.random(k) < 0.5, -vs, vs))
    inst = synth._build("uniform_check", n, kinds, [0] * m, lits)
    ctx = P.Context.from_instance(inst, device=0)
    s = ctx.search(100, seed=4)
    s.check()
    torch.cuda.synchronize()
    T = s.tensors()
    x = T["x"].cpu().numpy().astype(np.float64)
    Fo = oracle_of(inst)
    cnt, _, U = cdp.check(Fo, x, want_U=True)
    assert np.array_equal(T["unsat"].cpu().numpy(), cnt)
    assert np.array_equal(ctx.to_input_order(T["U"].cpu().numpy()), U)


@pytest.mark.parametrize("ks", [(129, 256, 257, 512), (513, 768, 769, 1024), (1025, 1280, 1281, 1536), (1537, 1792, 1793, 2048)])
def test_root_path_geometry_ladder(ks):
    """Cardinality constraints at every boundary of the root-path launch ladder (C, NW classes), fp64."""
    n = 2100
    rng = np.random.default_rng(sum(ks))
    kinds, bounds, lits = [], [], []
    for k in ks:
        vs = rng.choice(n, size=k, replace=False) + 1
        kinds.append(4); bounds.append(k // 3); lits.append(np.where(rng.random(k) < 0.5, -vs, vs))
        kinds.append(3); bounds.append(k // 2); lits.append(vs)
    inst = synth._build("ladder", n, kinds, bounds, lits)
    compare(inst, synth.points("U", 3, n, 31, np.float64), precision=64)
    compare(inst, synth.points("N", 2, n, 32, np.float64), precision=64)


@pytest.mark.parametrize("k", [128, 700, 2000])
def test_long_cardinality_fp32_probability_basis(k):
    """in the probability basis the fp32 root path stays within the fp32 tolerance (1e-4) even
    at k = 2000 (the ESP basis would fail at k ~ 32): forced precision 32, near-corner points."""
    n = k + 40
    rng = np.random.default_rng(k + 1)
    kinds, bounds, lits = [], [], []
    for kind, b in ((4, k // 4), (3, k // 2)):
        vs = rng.choice(n, size=k, replace=False) + 1
        kinds.append(kind); bounds.append(b); lits.append(np.where(rng.random(k) < 0.5, -vs, vs))
    inst = synth._build(f"fp32_long_k{k}", n, kinds, bounds, lits)
    compare(inst, synth.points("N", 8, n, 41), precision=32)
    compare(inst, synth.points("U", 8, n, 42), precision=32)


def test_maxsat_mode_planted_maxcut_tiny():
    """f3: optimisation mode (fixed weights, (RF)^inf, incumbent by falsified weight) finds the brute-force
    optimum of tiny planted Max-Cut instances (SPEC acceptance 7: >= 9 of 10 seeds)."""
    import itertools
    from paper_2308_15020_b200.maxsat import solve_maxsat
    hits = 0
    for seed in range(10):
        inst = synth.planted_maxcut(2, 4, seed=seed)
        Fo = oracle_of(inst)
        X = np.array(list(itertools.product((-1.0, 1.0), repeat=inst.n)))
        _, fw = cdp.check(Fo, X)
        ctx = P.Context.from_instance(inst, device=0)
        best, a, rounds, secs = solve_maxsat(ctx, batch=32, rounds=50, seed=seed, max_inner=50)
        assert ctx.check(a)[1] == best
        assert best >= fw.min() - 1e-12
        hits += abs(best - fw.min()) < 1e-9
    assert hits >= 9


@pytest.mark.parametrize("case", ["mixed", "long_card", "large_n", "large_n_long"])
def test_bit_packed_check_all_rules(case):
    """The round-end check (sign words of 32 points, OR / AND / parity reductions, bit-sliced counts for the
    other rules): unsat[b] and U_c (per constraint) bit-exact against the oracle's exact check, on a ragged
    batch with tie points (x = +-0 is False); large n reads the sign words without the shared tile."""
    if case == "mixed":
        inst = synth.random_mixed(n=150, m=900, seed=21, kmax=64)
    elif case == "long_card":
        inst = synth.config3(0, n=3000, m3=300, n_card=6, kmin=100, kmax=900)
    elif case == "large_n":
        inst = synth.random_mixed(n=40000, m=3000, seed=22, kmax=40)
    else:   # rows longer than 128 literals (check_long_kernel) with the sign words read without the shared tile
        inst = synth.config3(1, n=30000, m3=300, n_card=5, kmin=150, kmax=700)
    ctx = P.Context.from_instance(inst, device=0)
    B = 77
    s = ctx.search(B, seed=5)
    X = synth.points("Z", B, inst.n, 33, np.float64 if ctx.info["precision"] == 64 else np.float32)
    s.set_x(torch.from_numpy(X).cuda())
    s.check()
    torch.cuda.synchronize()
    T = s.tensors()
    Fo = oracle_of(inst)
    cnt, _, U = cdp.check(Fo, X.astype(np.float64), want_U=True)
    assert np.array_equal(T["unsat"].cpu().numpy(), cnt)
    assert np.array_equal(ctx.to_input_order(T["U"].cpu().numpy()), U)


@pytest.mark.parametrize("B", [7, 600, 1024, 1030])
def test_host_buffer_pipeline_matches_device(B):
    """Host-buffer evaluation (the public API with host pointers: staged in equal padded chunks, H2D / D2H
    overlapped with the chunk evaluations) against the oracle directly, and bit-identical to the device-buffer
    evaluation of the same batch (the launch plan is batch-independent), for ragged and exact chunk splits."""
    inst = synth.random_mixed(n=70, m=300, seed=14, kmax=40)
    X = synth.points("U", B, inst.n, 15)
    ctx, _, _ = compare(inst, X, device_path=False)
    fh, gh, uh = ctx.eval(X, grad=True, unsat=True)
    fd, gd, ud = ctx.eval(torch.from_numpy(X).cuda(), grad=True, unsat=True)
    assert np.array_equal(uh, ud.cpu().numpy())
    assert np.array_equal(fh, fd.cpu().numpy()) and np.array_equal(gh, gd.cpu().numpy())


@pytest.mark.parametrize("case,B", [("tiled", 600), ("tiled", 1024), ("tiled", 1030), ("global", 700),
                                    ("global_root", 520)])
def test_host_buffer_dual_stream_matches_device(case, B):
    """Host-buffer evaluation of >= 512 points: the batch splits into two half chunks evaluated concurrently on two
    compute streams, each with its own scratch and side streams (the global path's length-class groups and the
    root-path classes fork onto them); against the oracle, and bit-identical to the single-stream device-buffer
    evaluation."""
    if case == "tiled":
        inst = synth.random_ksat(n=120, m=3000, k=7, seed=23)
    elif case == "global":
        inst = synth.config4_hybrid(0, n=1024, m3=1500, n_xor=200, kmax=64)
    else:
        inst = synth.config3(0, n=1200, m3=2400, n_card=3, kmin=80, kmax=200)
    prec = 64 if case == "global_root" else 32
    X = synth.points("U", B, inst.n, 17, np.float64 if prec == 64 else np.float32)
    ctx, _, _ = compare(inst, X, device_path=False, precision=prec)
    assert ctx.info["path"] == (1 if case == "tiled" else 2)
    fh, gh, uh = ctx.eval(X, grad=True, unsat=True)
    fd, gd, ud = ctx.eval(torch.from_numpy(X).cuda(), grad=True, unsat=True)
    assert np.array_equal(uh, ud.cpu().numpy())
    assert np.array_equal(fh, fd.cpu().numpy()) and np.array_equal(gh, gd.cpu().numpy())


def test_host_buffer_nonfinite_rejected():
    """a non-finite coordinate in a host batch gives FFSAT_ERR_NONFINITE (flagged on the device)."""
    inst = synth.config1(0)
    ctx = P.Context.from_instance(inst, device=0)
    for bad in (np.nan, np.inf, -np.inf):
        X = synth.points("U", 700, inst.n, 16)
        X[613, 7] = bad
        with pytest.raises(P.FfsatError) as e:
            ctx.eval(X, grad=True)
        assert "NONFINITE" in str(e.value)
    f, g, _ = ctx.eval(synth.points("U", 700, inst.n, 16), grad=True)   # the context stays usable
    assert np.all(np.isfinite(f))
