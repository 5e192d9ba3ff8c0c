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
# replicate bench.py's timed loop (flush + per-step events + round end every 10 steps)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
T = s.tensors()
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
for use_flush in (True, False):
    evs = []
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for i in range(50):
        if use_flush: flush.zero_()
        a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        s.iterate(1)
        if (i + 1) % 10 == 0:
            s.check(); flag.copy_((T["unsat"].min() == 0).to(torch.int32).view(1)); s.restart(T["U"]); s.begin_round()
        a1.record(); evs.append((a0, a1))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    ev = [x.elapsed_time(y) for x, y in evs]
    print(f"bench loop flush={use_flush}: events mean {1e3*sum(ev)/len(ev):.1f} us/step (min {1e3*min(ev):.1f} max {1e3*max(ev):.1f}), wall {1e6*(t1-t0)/50:.1f} us/step")
