"""the paper's RQ1 gradient-timing suite (App. D) on one B200.

Seven random formulas (xor1-3, card1-3, xor+card; synth.rq1), 10 000 random points each ("average gradient
computation time per random point").  Per formula: the batched f + grad evaluation of all 10 000 points on the GPU
(device-resident buffers, CUDA events, median of 20 after warm-up) and through the public API with host buffers,
beside the CPU oracle (oracle/dp.c, fp64 GradSAT DP -- the paper's strongest CPU comparison, GradSAT, computes the
same DP) on the host cores.  Parity of the GPU results on these formulas is tests/test_parity_gpu.py::test_rq1_workloads.
The paper's own numbers are speedups of its A100 JAX implementation over 32-thread CPU solvers (1.2x on xor1 and
card1, 31.36x on xor3, 148.59x on card3): context, not a target.

Prints one JSON object per formula and writes them to the path given as argv[1] (default gpurun_out/rq1_suite.json).
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_15020_b200 as P  # noqa: E402
import synth  # noqa: E402
from oracle import cdp  # noqa: E402
from oracle.formula import OracleFormula  # noqa: E402

PAPER_SPEEDUP = {"xor1": 1.2, "card1": 1.2, "xor3": 31.36, "card3": 148.59}


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "rq1_suite.json")
    Bp = 10000
    rows = []
    for name in ("xor1", "xor2", "xor3", "card1", "card2", "card3", "xor+card"):
        inst = synth.rq1(name, seed=1)
        ctx = P.Context.from_instance(inst, device=0)
        dt = torch.float64 if ctx.info["precision"] == 64 else torch.float32
        X = synth.points("U", Bp, inst.n, 7, np.float64)
        xd = torch.from_numpy(X).to(dt).cuda()
        for _ in range(3):
            ctx.eval(xd)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.eval(xd)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        t_gpu = statistics.median(ts)
        xh = X.astype(np.float32 if dt == torch.float32 else np.float64)
        th = []
        for _ in range(5):
            t0 = time.perf_counter()
            ctx.eval(xh)
            th.append(time.perf_counter() - t0)
        t_host = statistics.median(th)
        Fo = OracleFormula.from_arrays(*inst.arrays())
        S = 500
        t0 = time.perf_counter()
        cdp.evaluate(Fo, X[:S])
        t_cpu = (time.perf_counter() - t0) / S * Bp
        row = {"formula": name, "n": inst.n, "m": inst.m, "literals": inst.n_lits, "points": Bp,
               "gpu_us_per_point": 1e6 * t_gpu / Bp, "gpu_e2e_us_per_point": 1e6 * t_host / Bp,
               "cpu_oracle_us_per_point": 1e6 * t_cpu / Bp, "cpu_threads": cdp.max_threads(),
               "speedup_vs_cpu_oracle": t_cpu / t_gpu, "paper_speedup_a100_vs_cpu": PAPER_SPEEDUP.get(name),
               "path": "tiled" if ctx.info["path"] == 1 else "global", "dtype": "f64" if dt == torch.float64 else "f32"}
        rows.append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    with open(out_path, "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
