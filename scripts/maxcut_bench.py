"""Benchmark-3-shaped weighted Max-Cut (planted partition) in optimisation mode on
one B200: p_t = 32 points, fixed weights, (RF)^inf, incumbent by falsified (uncut) weight; wall-clock cap
per instance.  Reports best cut weight found, rounds and seconds.  Writes argv[1] (JSON)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paper_2308_15020_b200 as P  # noqa: E402
import synth  # noqa: E402
from paper_2308_15020_b200.maxsat import solve_maxsat  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "maxcut_bench.json")
cap = float(sys.argv[2]) if len(sys.argv) > 2 else 5.0
rows = []
for l, k in ((16, 16), (16, 32), (32, 16), (32, 32)):
    for seed in range(2):
        inst = synth.planted_maxcut(l, k, seed)
        ctx = P.Context.from_instance(inst, device=0)
        best, a, rounds, secs = solve_maxsat(ctx, batch=32, rounds=10 ** 6, seed=seed, max_inner=100, timeout_s=cap)
        W = float(inst.weight.sum())
        cl = inst.meta["cluster"]
        row = {"l": l, "k": k, "seed": seed, "n": inst.n, "edges": inst.m, "total_weight": W, "best_uncut": best,
               "best_cut": W - best, "rounds": rounds, "seconds": secs}
        rows.append(row)
        print(json.dumps(row), flush=True)
os.makedirs(os.path.dirname(out), exist_ok=True)
json.dump(rows, open(out, "w"), indent=1)
