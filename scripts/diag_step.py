"""Diagnose bench step time: CPU enqueue cost vs GPU time per CLS iteration."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2308_15020_b200 as P, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
inst = {"c2": lambda: synth.config2(0), "c4": lambda: synth.config4_hybrid(0), "c3": lambda: synth.config3(0), "c5": lambda: synth.config5(0)}[cfg]()
B = {"c2": 1024, "c4": 1024, "c3": 32, "c5": 32}[cfg]
ctx = P.Context.from_instance(inst, device=0)
s = ctx.search(B, seed=1, max_inner=10**6)
s.begin_round(); torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N): s.iterate(1)
t1 = time.perf_counter()
torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"enqueue {1e6*(t1-t0)/N:.1f} us/iter, wall {1e6*(t2-t0)/N:.1f} us/iter")
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); s.iterate(N); e1.record(); torch.cuda.synchronize()
print(f"events around iterate({N}): {1e3*e0.elapsed_time(e1)/N:.1f} us/iter")
for what in ("check", "restart", "begin_round"):
    torch.cuda.synchronize(); e0.record()
    t0 = time.perf_counter()
    for _ in range(20): getattr(s, what)()
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
    print(f"{what}: enqueue {1e6*(t1-t0)/20:.1f} us, gpu {1e3*e0.elapsed_time(e1)/20:.1f} us")
