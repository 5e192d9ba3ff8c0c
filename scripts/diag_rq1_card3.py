"""Evaluate one RQ1 formula a few times on device buffers (for an ncu launch list)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2308_15020_b200 as P, synth
name = sys.argv[1] if len(sys.argv) > 1 else "card3"
inst = synth.rq1(name, seed=1)
ctx = P.Context.from_instance(inst, device=0)
xd = torch.from_numpy(synth.points("U", 10000, inst.n, 7, np.float32)).cuda()
for _ in range(6):
    ctx.eval(xd)
torch.cuda.synchronize()
print(ctx.info)
