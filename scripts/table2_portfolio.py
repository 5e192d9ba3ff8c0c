"""restart-heuristics study and portfolio in the shape of PAPER.md Table 2 on B200.

Instances: random 3-SAT at clause ratio 4.26, n in {50, 100, 150, 200, 250}; SATLIB's filtered-satisfiable uf sets
are an external dataset, so planted instances stand in (a hidden assignment makes them satisfiable; planted
instances are easier than filtered ones at the same ratio -- context only).  p_t = 1024 points per strategy, an
"iteration" is one restart round of 50 PGD steps (the rounded points are checked at its end), cap 1000 rounds; PAR-2
in rounds (unsolved = 2 x cap).  Variants, all through dist.solve_portfolio:
  w/o heuristics  fixed weights, a fresh random restart for every point (policy R),
  w/ heuristics   ERWA alpha = 0.4 + (ROF)^inf rephasing,
  portfolio       both at once (two searches of 1024 points on this GPU; on G GPUs the same code runs one strategy per
                  GPU group, dist.portfolio_groups) -- solved when either strategy solves.
Writes argv[1] (JSON)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_15020_b200 as P  # noqa: E402
from paper_2308_15020_b200 import dist as D  # noqa: E402
import synth  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "table2_portfolio.json")
per_n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cap, B, R = 1000, 1024, 50
STRATS = {"w/o heuristics": dict(policy="R", adaptive_weights=0), "w/ heuristics": dict(policy="ROF", adaptive_weights=1)}
torch.cuda.set_device(0)
rows = []
for n in (50, 100, 150, 200, 250):
    m = int(round(4.26 * n))
    res = {name: [] for name in list(STRATS) + ["portfolio"]}
    for i in range(per_n):
        z = np.random.default_rng(np.random.PCG64(10_000 + i)).random(n) < 0.5
        inst = synth.random_ksat(n, m, 3, seed=100 * n + i, planted=z)
        ctx = P.Context.from_instance(inst, device=0)
        for name, strats in [(k, [k]) for k in STRATS] + [("portfolio", list(STRATS))]:
            searches = [(j, ctx.search(B, seed=i, point0=list(STRATS).index(s) * B, max_inner=R, check_every=R,
                                       **STRATS[s]), None) for j, s in enumerate(strats)]
            r = D.solve_portfolio(searches, ctx.check, round_len=R, max_rounds=cap)
            ok = bool(r["sat"]) and ctx.check(r["assignment"])[0] == 0
            res[name].append((ok, r["rounds"], r["seconds"], strats[r["strategy"]] if ok and r["strategy"] >= 0 else None))
            for _, s, _ in searches:
                s.close()
        ctx.close()
    for name, rr in res.items():
        par2 = float(np.mean([rd if ok else 2 * cap for ok, rd, _, _ in rr]))
        row = {"n": n, "m": m, "variant": name, "instances": per_n, "solved": int(sum(ok for ok, *_ in rr)),
               "par2_rounds": par2, "median_seconds": float(np.median([t for _, _, t, _ in rr]))}
        if name == "portfolio":
            row["won_by"] = {k: sum(1 for ok, _, _, w in rr if ok and w == k) for k in STRATS}
        rows.append(row)
        print(json.dumps(row), flush=True)
os.makedirs(os.path.dirname(out), exist_ok=True)
json.dump({"note": "planted random 3-SAT at ratio 4.26 (SATLIB stand-in), p_t = 1024 per strategy, round = 50 PGD "
                   "steps, cap 1000 rounds, PAR-2 in rounds; paper Table 2 (P:1031-1037) is context",
           "rows": rows}, open(out, "w"), indent=1)
