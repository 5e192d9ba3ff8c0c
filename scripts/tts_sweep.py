"""Time-to-solve sweep over the clause ratio of planted random 7-SAT n=200 (1024 restart points)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2308_15020_b200 as P, synth
cap = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
for alpha in (30.0, 50.0, 65.0, 75.0, 87.79):
    inst = synth.config2(0, planted=True, alpha=alpha)
    ctx = P.Context.from_instance(inst, device=0)
    for mi in (50, 200):
        res, a = ctx.solve(batch=1024, max_restarts=100000, seed=1, max_inner=mi, check_every=10, timeout_s=cap)
        print(f"alpha={alpha} m={inst.m} max_inner={mi}: sat={res['sat']} check={ctx.check(a)[0]} t={res['seconds']:.2f}s "
              f"rounds={res['restarts']} iters={res['iterations']} best_unsat={res['best_unsat']}", flush=True)
