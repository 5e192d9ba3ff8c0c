"""CPU tests of the C-ABI library: it loads, exports every symbol include/ffsat.h declares, and its
host layer (parser, validation, classification, exact check) agrees with the oracle.  No compute
calls: host-only contexts (device = -1) refuse them."""
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden
import paper_2308_15020_b200 as P
from paper_2308_15020_b200 import build as B
from oracle import cdp
from oracle.formula import OracleFormula, parse
import synth


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def header_functions():
    txt = open(os.path.join(ROOT, "include", "ffsat.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ffsat_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 20
    out = subprocess.check_output(["nm", "-D", "--defined-only", P.LIB_PATH], text=True)
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    lib = P.lib()
    for n in names:
        assert hasattr(lib, n)
    assert set(P.EXPORTS) == set(names)


def test_library_is_sm100a():
    out = subprocess.check_output(["cuobjdump", "--list-elf", P.LIB_PATH], text=True)
    assert "sm_100a" in out


def _ctx(inst, **kw):
    return P.Context.from_instance(inst, device=-1, **kw)


def test_host_only_context_refuses_compute():
    c = _ctx(synth.config1(0))
    with pytest.raises(P.FfsatError) as e:
        c.eval(np.zeros((1, 20), np.float32))
    assert e.value.status == 1


@pytest.mark.parametrize("text,status,line", [
    ("p hnf 2 1\no 1 3 0\n", 3, 2), ("p hnf 2 1\no 1 -1 0\n", 4, 2), ("p hnf 3 2\no 1 0\nd 4 1 2 3 0\n", 5, 3),
    ("p hnf 2 1\no 1 2\n", 2, 2), ("o 1 0\n", 2, 1), ("p hnf 2 1\nq 1 0\n", 2, 2), ("p hnf 2 1\no 0\n", 2, 2),
    ("p whnf 2 1\nnan o 1 0\n", 6, 2), ("p cnf 2 1\n1 2\n", 2, 2)])
def test_parse_errors_carry_line(tmp_path, text, status, line):
    p = tmp_path / "f.hnf"
    p.write_text(text)
    with pytest.raises(P.FfsatError) as e:
        P.Context.from_file(str(p), device=-1)
    assert e.value.status == status
    assert f"line {line}" in str(e.value)


def test_parse_matches_oracle_parser(tmp_path):
    inst = synth.random_mixed(30, 80, 2, kmax=10)
    txt = inst.to_text(weighted=True)
    p = tmp_path / "f.whnf"
    p.write_text(txt)
    c = P.Context.from_file(str(p), device=-1)
    Fo = parse(txt)
    kind, bound, w, off, lits = c.export()
    assert np.array_equal(kind, Fo.kind) and np.array_equal(bound, Fo.bound)
    assert np.array_equal(off, Fo.offsets) and np.array_equal(lits, Fo.lits) and np.allclose(w, Fo.weight)
    for name in ("eg2_eg3_card4_ge2.hnf", "eg7_saddle.hnf", "eg8_local.hnf"):
        c = P.Context.from_file(golden(name), device=-1)
        Fo = parse(open(golden(name)).read())
        assert np.array_equal(c.export()[4], Fo.lits)


def test_array_validation():
    with pytest.raises(P.FfsatError) as e:
        P.Context.from_arrays(3, [3], [5], None, [0, 2], [1, 2], device=-1)
    assert e.value.status == 5
    with pytest.raises(P.FfsatError) as e:
        P.Context.from_arrays(3, [0], None, [float("inf")], [0, 2], [1, 2], device=-1)
    assert e.value.status == 6
    with pytest.raises(P.FfsatError) as e:
        P.Context.from_arrays(3, [0], None, None, [0, 0], [], device=-1)
    assert e.value.status == 1


def test_classification_counts():
    """OR/XOR/XNOR/NAE and the degenerate cardinalities take the product fast path (F3); other
    cardinalities and any constraint with k > 64 take the root path."""
    cons = [(0, 0, 1.0, [1, 2, 3]), (1, 0, 1.0, [1, 2]), (2, 0, 1.0, [3, 4]), (5, 0, 1.0, [1, 2, 3]),
            (3, 1, 1.0, [1, 2]), (3, 0, 1.0, [1, 2]), (3, 3, 1.0, [1, 2, 3]), (4, 0, 1.0, [1, 2]), (4, 1, 1.0, [1, 2]),
            (4, 2, 1.0, [1, 2]), (3, 2, 1.0, [1, 2, 3]), (4, 1, 1.0, [1, 2, 3])]
    long_or = list(range(1, 81))
    cons.append((0, 0, 1.0, long_or))
    Fo = OracleFormula.from_constraints(80, cons)
    c = P.Context.from_arrays(80, Fo.kind, Fo.bound, Fo.weight, Fo.offsets, Fo.lits, device=-1)
    assert c.info["n_fast_cons"] == 10 and c.info["n_sym_cons"] == 3
    assert c.info["precision"] == 64  # a root-path constraint longer than 64


def test_exact_check_matches_oracle():
    for inst in (synth.random_mixed(25, 120, 5, kmax=12), synth.config4_parity(1), synth.config1(2)):
        c = _ctx(inst)
        Fo = OracleFormula.from_arrays(*inst.arrays())
        X = synth.points("C", 64, inst.n, 9, np.float64)
        cnt, fw = cdp.check(Fo, X)
        for b in range(64):
            a = np.where(X[b] < 0, -1, 1).astype(np.int8)
            n_u, w_u = c.check(a)
            assert n_u == cnt[b] and abs(w_u - fw[b]) < 1e-12


def test_paths_and_sizes():
    small = _ctx(synth.config2(0))
    assert small.info["path"] == 1 and small.info["precision"] == 32
    assert small.info["n_lits"] == 7 * 17000
    c3 = _ctx(synth.config3(0, n=4096, m3=100, n_card=2, kmin=500, kmax=600))
    assert c3.info["path"] == 2 and c3.info["precision"] == 64 and c3.info["n_sym_cons"] == 2


@pytest.mark.parametrize("maker", [lambda: synth.config2(0), lambda: synth.config1(2),
                                   lambda: synth.random_mixed(n=120, m=600, seed=3, kmax=16),
                                   lambda: synth.rq1("xor2", seed=1)])
def test_tiled_units_are_var_disjoint_classes(maker):
    """The tiled kernels add a unit's literal terms into the shared gradient tile from 8 warps at once; that is
    race-free and deterministic only because no variable occurs twice in a unit (host: disjoint_classes).
    Also: units cover every fast constraint exactly once, in position order, with <= 16 members."""
    inst = maker()
    ctx = P.Context.from_instance(inst, device=-1)
    assert ctx.info["path"] == 1
    units, order = ctx.layout_units()
    assert sorted(order.tolist()) == list(range(inst.m))
    covered = 0
    for bucket, count, p0, tiled in units:
        assert tiled == 1 and 1 <= count <= 16 and p0 == covered
        seen = set()
        for p in range(p0, p0 + count):
            c = order[p]
            vs = np.abs(inst.lits[inst.offsets[c]:inst.offsets[c + 1]])
            assert not (seen & set(vs.tolist())), "variable shared inside a unit"
            seen |= set(vs.tolist())
        covered += count
    assert covered == ctx.info["n_fast_cons"]


@pytest.mark.parametrize("maker", [lambda: synth.config4_hybrid(0), lambda: synth.random_mixed(n=900, m=700, seed=5, kmax=64)])
def test_global_units_length_classes(maker):
    """Global path: units are runs of one bucket in position order covering every fast constraint once, buckets
    ascend in k so the length classes the kernels split on (k <= 4, 4 < k <= 16, k > 16: the long kernel) are
    contiguous unit ranges, and a unit holds <= max(1, cap / k) constraints (cap in 32..512 literals)."""
    inst = maker()
    ctx = P.Context.from_instance(inst, device=-1, path=2)
    assert ctx.info["path"] == 2
    units, order = ctx.layout_units()
    assert sorted(order.tolist()) == list(range(inst.m))
    k_of = np.diff(inst.offsets)
    covered, last_cls, last_k = 0, -1, 0
    for bucket, count, p0, tiled in units:
        assert tiled == 0 and p0 == covered and count >= 1
        ks = {int(k_of[order[p]]) for p in range(p0, p0 + count)}
        assert len(ks) == 1
        k = ks.pop()
        assert count <= max(1, 512 // k)
        assert k >= last_k
        cls = 0 if k <= 4 else 1 if k <= 16 else 2
        assert cls >= last_cls
        last_cls, last_k = cls, k
        covered += count
    assert covered == ctx.info["n_fast_cons"]


def test_product_tree_classification(monkeypatch):
    """fp64 symmetric constraints of 256..2048 literals take the product-tree path (ffsat_info n_tree_cons, its FP64
    instruction count tree_work, the root path's k M' count sym_root_lits only for the others); FFSAT_TREE=0 keeps
    them on the root path; fp32 contexts never use the tree."""
    inst = synth.config3(0, n=3000, m3=50, n_card=4, kmin=300, kmax=2000)
    c = _ctx(inst)
    assert c.info["n_tree_cons"] == 4 and c.info["tree_work"] > 0 and c.info["sym_root_lits"] == 0
    ks = [len(set(inst.lits[inst.offsets[i]:inst.offsets[i + 1]])) for i in range(inst.m - 4, inst.m)]
    # the tree's FP64 count is far below the root path's 12 k M' (about k^2 / 1.3 vs 6 k^2)
    assert c.info["tree_work"] < sum(12 * k * ((k + 1) // 2) for k in ks) / 5
    monkeypatch.setenv("FFSAT_TREE", "0")
    r = _ctx(inst)
    assert r.info["n_tree_cons"] == 0 and r.info["sym_root_lits"] == sum(k * ((k + 1) // 2) for k in ks)
    monkeypatch.delenv("FFSAT_TREE")
    f32 = P.Context.from_instance(inst, precision=32, device=-1)
    assert f32.info["n_tree_cons"] == 0


def test_solve_params_defaults_and_fista_flag():
    """ffsat_default_params: the documented defaults, accel = 0 (monotone Armijo, reading #16); accel = 1
    selects FISTA (reading #16b)."""
    p = P.ffsat_default_params()
    assert (p.eta0, p.eta_min, p.armijo_c1, p.alpha, p.max_inner, p.check_every, p.policy, p.adaptive_weights) == \
        (1.0, 1e-12, 1e-4, 0.4, 500, 10, 0, 1)
    assert p.accel == 0 and p.reserved == 0
    assert P.ffsat_default_params(accel=1).accel == 1
