"""restart-heuristics ablation in the shape of PAPER.md Table 2 on one B200.

Instances: random 3-SAT at clause ratio 4.26, n in {50, 100, 150, 200, 250}; SATLIB's filtered-satisfiable uf
sets are an external dataset, so planted instances stand in (a hidden assignment makes them satisfiable; planted
instances are easier than filtered ones at the same ratio -- context only).  p_t = 1024 points, an "iteration" is
one restart round of 50 PGD steps, cap 1000 rounds; PAR-2 in rounds (unsolved = 2 x cap).  Variants: heuristics
on (ERWA alpha = 0.4 + (ROF)^inf rephasing) and off (fixed weights, fresh random restarts only).
Writes argv[1] (JSON)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paper_2308_15020_b200 as P  # noqa: E402
import synth  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "table2.json")
per_n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cap_rounds = 1000
rows = []
for n in (50, 100, 150, 200, 250):
    m = int(round(4.26 * n))
    for name, params in (("heuristics", dict(policy="ROF", adaptive_weights=1)), ("none", dict(policy="R", adaptive_weights=0))):
        rounds, solved, secs = [], 0, []
        for i in range(per_n):
            z = np.random.default_rng(np.random.PCG64(10_000 + i)).random(n) < 0.5
            inst = synth.random_ksat(n, m, 3, seed=100 * n + i, planted=z)
            ctx = P.Context.from_instance(inst, device=0)
            res, a = ctx.solve(batch=1024, max_restarts=cap_rounds, seed=i, max_inner=50, check_every=10, **params)
            ok = bool(res["sat"]) and ctx.check(a)[0] == 0
            solved += ok
            rounds.append(res["restarts"] if ok else 2 * cap_rounds)
            secs.append(res["seconds"])
        row = {"n": n, "m": m, "variant": name, "instances": per_n, "solved": solved, "par2_rounds": float(np.mean(rounds)),
               "median_seconds": float(np.median(secs))}
        rows.append(row)
        print(json.dumps(row), flush=True)
os.makedirs(os.path.dirname(out), exist_ok=True)
json.dump(rows, open(out, "w"), indent=1)
