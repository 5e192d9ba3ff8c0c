"""precision of the root-of-unity path in the probability basis, fp32 vs fp64, up to k = 2000.

For each length k: two at-most / at-least constraints over random literals, 16 uniform and 16 near-corner points
(|x| = 1 - U(0, 1e-3), the late-PGD regime where the ESP basis cancels catastrophically); the GPU root
path forced to fp32 and to fp64, each compared with the fp64 oracle (GradSAT DP) on exactly the values the GPU saw.
Reports the worst relative error max |d| / max(1, |ref|) of f and of the gradient.  Writes argv[1] (JSON).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2308_15020_b200 as P  # noqa: E402
import synth  # noqa: E402
from oracle import cdp  # noqa: E402
from oracle.formula import OracleFormula  # noqa: E402


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "precision_study.json")
    rows = []
    for k in (16, 32, 64, 128, 256, 500, 1000, 2000):
        n = 2 * k + 8
        rng = np.random.default_rng(k)
        kinds, bounds, lits = [], [], []
        for kind, b in ((4, k // 4), (3, k // 2)):
            vs = rng.choice(n, size=k, replace=False) + 1
            kinds.append(kind); bounds.append(b); lits.append(np.where(rng.random(k) < 0.5, -vs, vs))
        inst = synth._build(f"prec_k{k}", n, kinds, bounds, lits)
        Fo = OracleFormula.from_arrays(*inst.arrays())
        row = {"k": k}
        for prec, dt in ((32, np.float32), (64, np.float64)):
            ctx = P.Context.from_instance(inst, precision=prec, device=0)
            worst_f = worst_g = 0.0
            for dist, seed in (("U", 1), ("N", 2)):
                X = synth.points(dist, 16, n, seed, dt)
                f, g, _ = ctx.eval(X)
                fo, go = cdp.evaluate(Fo, X.astype(np.float64))
                worst_f = max(worst_f, float(np.max(np.abs(f - fo) / np.maximum(1, np.abs(fo)))))
                worst_g = max(worst_g, float(np.max(np.abs(g - go) / np.maximum(1, np.abs(go)))))
            row[f"fp{prec}_f_err"] = worst_f
            row[f"fp{prec}_grad_err"] = worst_g
        rows.append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    with open(out_path, "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
