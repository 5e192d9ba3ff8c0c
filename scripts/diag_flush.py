"""Per-step event times of the bench loop under different L2-flush methods."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2308_15020_b200 as P, synth
inst = synth.config2(0)
ctx = P.Context.from_instance(inst, device=0)
s = ctx.search(1024, seed=1, max_inner=10**6)
s.begin_round(); torch.cuda.synchronize()
buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
sink = torch.empty(1, dtype=torch.float32, device="cuda")
methods = {"none": lambda: None, "zero_256M": lambda: buf.zero_(), "fill_256M": lambda: buf.fill_(1.0),
           "read_256M": lambda: torch.sum(buf, dim=0, out=sink[0]) if False else sink.copy_(buf.sum().view(1)),
           "zero_160M": lambda: buf[: 160 * 1024 * 1024 // 4].zero_()}
for name, fl in methods.items():
    for rep in range(2):
        evs = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(60):
            fl()
            a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
            a0.record(); s.iterate(1); a1.record(); evs.append((a0, a1))
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / 60
        ev = np.array([x.elapsed_time(y) for x, y in evs]) * 1e3
        print(f"{name:10s} rep{rep}: median {np.median(ev):7.1f} mean {ev.mean():8.1f} max {ev.max():8.1f} us; wall {wall*1e6:7.1f} us/step; "
              f">1ms: {[(i, round(v)) for i, v in enumerate(ev) if v > 1000]}")
# flush kernel alone
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): buf.zero_()
e1.record(); torch.cuda.synchronize(); print(f"zero_256M alone: {e0.elapsed_time(e1)/20*1e3:.1f} us")
