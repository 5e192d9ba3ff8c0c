"""Solver-parameter sweep for time-to-solve on planted random 7-SAT n=200 (1024 points)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_15020_b200 as P, synth
cap = float(sys.argv[1]) if len(sys.argv) > 1 else 6.0
for alpha in (75.0, 87.79):
    inst = synth.config2(0, planted=True, alpha=alpha)
    ctx = P.Context.from_instance(inst, device=0)
    for mi, eta0, pol, alp in ((200, 1.0, "ROF", 0.4), (50, 1.0, "ROF", 0.4), (1000, 1.0, "ROF", 0.4), (200, 4.0, "ROF", 0.4),
                               (200, 16.0, "ROF", 0.4), (200, 1.0, "RF", 0.4), (200, 1.0, "ROF", 0.1), (200, 1.0, "ROF", 0.8)):
        res, a = ctx.solve(batch=1024, max_restarts=10 ** 6, seed=1, max_inner=mi, check_every=10, eta0=eta0, policy=pol,
                           alpha=alp, timeout_s=cap)
        print(json.dumps({"alpha": alpha, "max_inner": mi, "eta0": eta0, "policy": pol, "erwa_alpha": alp, "sat": res["sat"],
                          "check": int(ctx.check(a)[0]), "best_unsat": res["best_unsat"], "s": round(res["seconds"], 2),
                          "rounds": res["restarts"]}), flush=True)
