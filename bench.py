#!/usr/bin/env python
"""bench.py -- FastFourierSAT hot path on B200 (BASELINE.json metric: literal-gradient terms/s).

Default workload = BASELINE.json configs[1] (c2): uniform random 7-SAT, n = 200, m = 17000
(alpha = 85), a batch of 1024 restart points per GPU, the full projected-gradient CLS loop.

One *step* = one CLS iteration over the batch (every row of SURVEY.md 8(a) on the hot path):
  A4-A7  one batched f + grad evaluation at the trial points (gather, products, deterministic reductions),
         with the fused A9 sign check of the trial points,
  A8     the Armijo accept / eta update / next projected trial point,
and every --round-len steps the round end: A9 exact check of sgn(x) (unsat[b], U_c), A11 the
restart-sharding collectives (U_c SUM and any-solved MAX over ranks, NCCL), A10 ERWA + rephase,
and the next round's start evaluation.  A1-A3 (parse, layout, coefficients) run once at load.

value = literal-gradient terms per second over all ranks = sum_c k_c * B_total * K / t, with t the
max over ranks of the summed CUDA-event step times (L2 flushed between steps, untimed).
`--impl reference` times the oracle (oracle/dp.c, the CPU fp64 GradSAT DP) on the same workload.

`python bench.py --gpus N` without a torchrun environment re-executes itself under torch.distributed.run with N
ranks (127.0.0.1); with fewer visible GPUs than ranks the ranks share devices over gloo (a functional dry run).

roofline: every resource the dominant kernel (or, for HBM, the evaluation)
uses is reported under "resources" with its algorithmic count -- fast paths 3 products per term (FP32 pipe) and
12 B per term of shared-memory traffic on the on-chip path, the root path 12 FP64 slots per (literal, root), HBM
4L + 8C + 2 es n B + 4B bytes per evaluation -- and the top-level entry is the BINDING one (highest fraction).
traffic = ncu dram bytes of the same scope; waste = traffic / algorithmic bytes.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

# mode "restart": a step is one CLS iteration of the batch, restart points sharded over ranks (weak scaling);
# mode "constraint": a step is one batched f + grad evaluation, constraints sharded over ranks + all-reduce
CONFIGS = {
    "c2": dict(make=lambda: synth.config2(0), B=1024, mode="restart", desc="c2: uniform random 7-SAT n=200 m=17000 (alpha=85)"),
    "c1": dict(make=lambda: synth.config1(0), B=1, mode="restart", desc="c1: uniform random 3-SAT n=20 m=91, single point"),
    "c3": dict(make=lambda: synth.config3(0), B=32, mode="restart", desc="c3: n=4096, 8192 planted 3-SAT + 32 at-most-b k=500..2000, fp64"),
    "c3b256": dict(make=lambda: synth.config3(0), B=256, mode="restart", desc="c3 at B=256: n=4096, 8192 planted 3-SAT + 32 at-most-b k=500..2000, fp64"),
    "c4p": dict(make=lambda: synth.config4_parity(0), B=1024, mode="restart", desc="c4(i): parity learning with error N=60, m=120 XOR (P:1066-1071)"),
    "c4": dict(make=lambda: synth.config4_hybrid(0), B=1024, mode="restart", desc="c4: n=1024, 2048 planted 3-CNF + 512 XOR k=3..64"),
    "c5": dict(make=lambda: synth.config5(0), B=32, mode="constraint", desc="c5: uniform random 3-SAT n=1e6 m=4.2e6, constraint-sharded"),
    "c5b1": dict(make=lambda: synth.config5(0), B=1, mode="constraint", desc="c5 at B=1: uniform random 3-SAT n=1e6 m=4.2e6, one point"),
}
SM_COUNT = 148
FP32_LANES, FP64_LANES = 128, 64  # FP32 / FP64 lanes per SM per clock (B200 guide unit counts)
# Algorithmic FP lane-operations (one FMA = one lane-op = one pipe slot: count instructions):
SMEM_BYTES_PER_TERM = 12   # x tile LDS + gradient tile LDS + STS, 4 B each
TMEM_RMW_BYTES_PER_CLK = 213   # per SM: 16 warps of 32x32b.x2 tcgen05.ld + tcgen05.st (profiles/r02_tmem_probe.txt)
FAST_PRODUCTS_PER_TERM = 3       # the fast-path product count per literal and point (prefix, suffix, term)
ROOT_OPS_PER_LIT_ROOT = 12        # factor 2 FMA, prefix + suffix complex MUL (2 x 4), Re-accumulate 2 FMA (App. A)


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled every `interval` s during the timed region through NVML
    (in-process; nvidia-smi polling was measured to stall kernel launches)."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, dev, interval=0.1):
        self.dev, self.interval = dev, interval
        self.samples = []
        self.stop_ev = threading.Event()
        self.t = None
        self.err = None

    def start(self):
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            idx = torch.cuda._get_nvml_device_index(self.dev) if hasattr(torch.cuda, "_get_nvml_device_index") else self.dev
            self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv, h = self.nv, self.h
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_ev.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), int(get_reasons(h))))
            except Exception:  # noqa: BLE001
                pass
            self.stop_ev.wait(self.interval)

    def stop(self):
        if self.t is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "not sampled"]}
        self.stop_ev.set()
        self.t.join()
        sm = [c for c, _ in self.samples]
        reasons = sorted({nm for _, r in self.samples for bit, nm in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax, "reasons": reasons,
                "samples": len(sm), "source": "nvml"}


def ncu_traffic(kernel_key, config, any_of=False):
    """dram bytes per launch of the dominant kernel(s) ("a+b": summed) on this config from the committed ncu summary
    (profiles/ncu_summary.json, keys "<config>:<kernel>" per launch of one evaluation), or None.  any_of: sum the
    kernels present (an evaluation launches a subset of them), None if none is."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as fh:
            d = json.load(fh)
        vals = [d.get(f"{config}:{k}", {}).get("dram_bytes_per_launch") for k in kernel_key.split("+")]
        if any_of:
            vals = [v for v in vals if v is not None]
            return float(sum(vals)) if vals else None
        return None if any(v is None for v in vals) else float(sum(vals))
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------------------------------------------ reference arm


def run_reference(args, cfg, inst):
    """The oracle (oracle/dp.c, fp64 CPU GradSAT DP, OpenMP over points) as it stands, on the same workload:
    each step evaluates f and grad on a bounded sample of the workload's points."""
    from oracle import cdp
    from oracle.formula import OracleFormula
    Fo = OracleFormula.from_arrays(*inst.arrays())
    threads = cdp.max_threads()
    X = synth.points("U", cfg["B"], inst.n, 1000, np.float64)
    t0 = time.perf_counter()
    cdp.evaluate(Fo, X[:1])
    one = time.perf_counter() - t0
    budget = max(0.05, 150.0 / max(1, args.steps + args.warmup))  # whole run within ~3 minutes
    S = int(max(1, min(cfg["B"], budget / max(one / max(1, threads), 1e-6))))
    Xs = X[:S]
    for _ in range(args.warmup):
        cdp.evaluate(Fo, Xs)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cdp.evaluate(Fo, Xs)
        ts.append(time.perf_counter() - t0)
    t = sum(ts)
    L = inst.n_lits
    value = L * S * args.steps / t
    sample = f"{S} of the {cfg['B']} points per step (fp64 f + grad), {threads} OpenMP threads"
    line = {"impl": "reference", "metric": "literal-gradient terms/s", "value": value, "unit": "terms/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "points_per_step": S},
            "cpu_baseline": {"value": value, "unit": "terms/s", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "terms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, inst, X):
    """Oracle timed on the host cores on a bounded sample (SURVEY 8(d) oracle timing): three timed runs of ~3.5 s each
    (the sample repeated until then), median of the three rates; plus a 1-thread rate and the host CPU model."""
    import platform
    import subprocess
    from oracle import cdp
    from oracle.formula import OracleFormula
    Fo = OracleFormula.from_arrays(*inst.arrays())
    threads = cdp.max_threads()
    Xd = X.astype(np.float64)
    t0 = time.perf_counter()
    cdp.evaluate(Fo, Xd[:min(len(Xd), threads)])
    probe = time.perf_counter() - t0
    per_pt = probe / min(len(Xd), threads) * threads  # wall per point per thread-batch
    S = int(max(1, min(len(Xd), 3.5 / max(per_pt / threads, 1e-9))))
    rates, reps_all = [], []
    for _ in range(3):
        reps, t0 = 0, time.perf_counter()
        while True:
            cdp.evaluate(Fo, Xd[:S])
            reps += 1
            t = time.perf_counter() - t0
            if t >= 3.5 or reps >= 1000:
                break
        rates.append(inst.n_lits * S * reps / t)
        reps_all.append(reps)
    # the 1-thread rate on a smaller sample (SURVEY 8(d) oracle timing) and the host CPU model
    S1 = int(max(1, min(S, 2.0 / max(per_pt, 1e-9))))
    t0 = time.perf_counter()
    cdp.evaluate(Fo, Xd[:S1], threads=1)
    t1 = time.perf_counter() - t0
    cpu = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        cpu = next((ln.split(":", 1)[1].strip() for ln in out.splitlines() if ln.startswith("Model name")), "")
        sockets = next((ln.split(":", 1)[1].strip() for ln in out.splitlines() if ln.startswith("Socket(s)")), "")
        cpu = f"{cpu} ({sockets} socket(s), {os.cpu_count()} logical CPUs, {platform.machine()})"
    except (OSError, subprocess.SubprocessError, StopIteration):
        pass
    return {"value": float(statistics.median(rates)), "unit": "terms/s", "cores": threads, "kind": "oracle",
            "sample": f"f + grad of {S} of the workload's {len(Xd)} points in fp64, repeated for 3.5 s, median of 3 runs "
                      f"({reps_all} repetitions)",
            "runs": rates, "value_1_thread": inst.n_lits * S1 / t1, "sample_1_thread": f"{S1} points ({t1:.1f} s)", "cpu": cpu}


# ------------------------------------------------------------------------------------------------ our arm


def time_to_solve(P, D, args, device, rank, world, dist):
    """BJ.metric time-to-solve on G = world GPUs: restart-sharded Alg. 1 (dist.solve_sharded: every rank
    runs 1024 restart points, the ranks exchange U_c and the library's any-solved / incumbent keys at each round end
    and stop together on the first verified solution) on planted c2 instances (random 7-SAT n=200 with a hidden
    satisfying assignment) at the threshold ratio alpha = 87.79 and at alpha = 65; ERWA + (ROF) rephasing, 200 PGD
    trials per round, any-solved polled every 10 iterations.  Wall time of rank 0 from the first iteration to the
    verified answer, one run per seed; median and PAR-2 (an unsolved run counts 2 x cap)."""
    import torch
    out = []
    for alpha in (87.79, 65.0):
        inst = synth.config2(0, planted=True, alpha=alpha)
        ctx = P.Context.from_instance(inst, device=device)
        times, solved, rounds, best = [], 0, [], []
        for seed in range(-1, args.tts_seeds):                 # seed -1: untimed warm-up (module loading)
            s = ctx.search(1024, seed=1 + max(seed, 0), point0=rank * 1024, max_inner=200, check_every=200)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            r = D.solve_sharded(s, ctx.check, round_len=200, max_rounds=10 ** 6 if seed >= 0 else 1, rank=rank,
                                world=world, timeout_s=args.tts_cap if seed >= 0 else 0.0, poll_every=10)
            s.close()
            if seed < 0:
                continue
            ok = bool(r["sat"]) and ctx.check(r["assignment"])[0] == 0
            solved += ok
            times.append(r["seconds"] if ok else 2 * args.tts_cap)
            rounds.append(r["rounds"])
            best.append(int(r["best_unsat"]))
        out.append({"instance": f"planted 7-SAT n={inst.n} m={inst.m} (alpha {alpha})", "batch_per_gpu": 1024,
                    "batch_total": 1024 * world, "gpus": world, "seeds": args.tts_seeds, "solved": solved,
                    "cap_s": args.tts_cap, "median_s": float(np.median(times)), "par2_s": float(np.mean(times)),
                    "seconds": times, "restart_rounds": rounds, "best_unsat": best})
        ctx.close()
    return {"runs": out, "note": "dist.solve_sharded over all ranks; sat only after the exact host check "
                                 "(ffsat_check); unsolved = 2 x cap"}


def roofline_of(info, inst, B, ph, args):
    """Every resource the hot path uses, with SURVEY 8(d)'s algorithmic counts, and the binding one."""
    peaks, peak_src = measured_peaks()
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    fast_ms, root_ms = float(ph[0]), float(ph[1])
    eval_ms = float(np.sum(ph))
    f64 = info["precision"] == 64
    es = 8 if f64 else 4
    terms_fast = info["n_fast_lits"] * B
    L, C, n = inst.n_lits, inst.m, inst.n
    alg_bytes = 4 * L + 8 * C + 2 * es * n * B + 4 * B
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    lanes = FP64_LANES if f64 else FP32_LANES
    alu_peak = SM_COUNT * lanes * mhz * 1e6 / 1e12
    alu_src = (f"{SM_COUNT} SMs x {lanes} {'FP64' if f64 else 'FP32'} lanes x {mhz:.0f} MHz ({peak_src} sm_max_mhz); "
               "one FMA / MUL = one lane-op")
    res = {}
    eval_kernels = ("transpose_kernel+canon_copy_kernel+fast_global_kernel+fast_global_long_kernel+owner_grad_kernel+owner_grp_kernel+"
                    "fold_rows_kernel+reduce_grad_kernel+reduce_f_kernel"
                    if info["path"] == 2 else "fast_wide_kernel+fast_tiled_kernel+reduce_grad_kernel+reduce_f_kernel")
    traffic_eval = ncu_traffic(eval_kernels, args.config, any_of=True)
    res["hbm"] = {"scope": "evaluation (A4-A7, every kernel)", "achieved": alg_bytes / (eval_ms * 1e-3) / 1e9,
                  "peak": hbm_peak, "unit": "GB/s", "algorithmic_bytes": alg_bytes,
                  "algorithmic_def": f"4L + 8C + 2*{es}*n*B + 4B (SURVEY 8(d))", "time_ms": eval_ms,
                  "traffic": traffic_eval, "waste": (traffic_eval / alg_bytes) if traffic_eval else None,
                  "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}
    grad_ms = float(ph[2])
    own = info.get("n_own_lits", 0) > 0
    if own and grad_ms >= max(fast_ms, root_ms):
        # global path, owner-computes: the short constraints' products are formed in the owner kernel (grouped
        # records when they are the only fast constraints, owner_grp_kernel; else owner_grad_kernel)
        oname = "owner_grp_kernel" if info["n_own_lits"] == info["n_fast_lits"] else "owner_grad_kernel"
        res["alu"] = {
            "scope": oname, "pipe": "fp64" if f64 else "fp32",
            "achieved": FAST_PRODUCTS_PER_TERM * terms_fast / (grad_ms * 1e-3) / 1e12, "peak": alu_peak,
            "unit": "T lane-op/s", "algorithmic_def": f"{FAST_PRODUCTS_PER_TERM} products per literal term (SURVEY 8(d))",
            "time_ms": grad_ms, "peak_source": alu_src}
        kms = grad_ms
    elif fast_ms >= root_ms:
        kname = ("fast_global_kernel+fast_global_long_kernel" if info["path"] == 2 else
                 "fast_tmem_kernel" if info.get("wide") == 2 else
                 "fast_wide_kernel" if info.get("wide") else "fast_tiled_kernel")
        res["alu"] = {
            "scope": kname, "pipe": "fp64" if f64 else "fp32", "achieved": FAST_PRODUCTS_PER_TERM * terms_fast / (fast_ms * 1e-3) / 1e12, "peak": alu_peak,
            "unit": "T lane-op/s", "algorithmic_def": f"{FAST_PRODUCTS_PER_TERM} products per literal term (SURVEY 8(d))",
            "time_ms": fast_ms, "peak_source": alu_src}
        if info["path"] == 1:
            smem_peak = SM_COUNT * 128 * mhz * 1e6 / 1e9
            tm = info.get("wide") == 2
            sb = 4 if tm else SMEM_BYTES_PER_TERM
            res["smem"] = {"scope": kname, "achieved": sb * terms_fast / (fast_ms * 1e-3) / 1e9,
                           "peak": smem_peak, "unit": "GB/s",
                           "algorithmic_def": (f"{sb} B per term: x tile read" if tm else
                                               f"{sb} B per term: x tile read + gradient tile read and write"),
                           "time_ms": fast_ms, "peak_source": f"{SM_COUNT} SMs x 128 B/clk x {mhz:.0f} MHz"}
            if tm:
                tmem_peak = SM_COUNT * TMEM_RMW_BYTES_PER_CLK * mhz * 1e6 / 1e9
                res["tmem"] = {"scope": kname, "achieved": 8 * terms_fast / (fast_ms * 1e-3) / 1e9, "peak": tmem_peak,
                               "unit": "GB/s", "algorithmic_def": "8 B per term: gradient tile read and write in TMEM",
                               "time_ms": fast_ms,
                               "peak_source": f"{SM_COUNT} SMs x {TMEM_RMW_BYTES_PER_CLK} B/clk (tcgen05.ld + st read-modify-"
                                              f"write, measured by scripts/tmem_probe.cu) x {mhz:.0f} MHz"}
        kms = fast_ms
    else:
        # root phase: the product-tree kernel (long fp64 constraints: its own FP64 instruction count, tree_work) and the
        # root-of-unity kernels (12 slots per (literal, root)) for the rest
        tree = info.get("n_tree_cons", 0) > 0
        kname = "+".join((["sym_tree_kernel"] if tree else []) + (["sym_item_kernel"] if info["sym_root_lits"] else []))
        kms = root_ms
        ops = ROOT_OPS_PER_LIT_ROOT * info["sym_root_lits"] + info.get("tree_work", 0)
        res["alu"] = {
            "scope": kname, "pipe": "fp64" if f64 else "fp32", "achieved": ops * B / (root_ms * 1e-3) / 1e12,
            "peak": alu_peak, "unit": "T lane-op/s",
            "algorithmic_def": ((f"product tree: {info['tree_work']} FP64 instructions per point (one per multiply-add of the "
                                 f"level convolutions / correlations, leaf recurrences; tree::tree_fp64_work)" if tree else "") +
                                (" + " if tree and info["sym_root_lits"] else "") +
                                (f"{ROOT_OPS_PER_LIT_ROOT} slots per (literal, root) (SURVEY App. A)" if info["sym_root_lits"] else "")),
            "time_ms": root_ms, "peak_source": alu_src}
    for r in res.values():
        r["frac"] = r["achieved"] / r["peak"]
    bound = max(res, key=lambda k: res[k]["frac"])
    top = res[bound]
    traffic = top.get("traffic") if bound == "hbm" else ncu_traffic(top["scope"], args.config)
    return {"bound": bound, "achieved": top["achieved"], "peak": top["peak"], "unit": top["unit"], "frac": top["frac"],
            "traffic": traffic, "kernel": top["scope"], "kernel_ms": top["time_ms"],
            "waste": res["hbm"]["waste"], "resources": res,
            "eval_phase_ms": {"fast": float(ph[0]), "root": float(ph[1]), "grad_reduce": float(ph[2]), "f_reduce": float(ph[3])},
            "kernel_share_of_eval": kms / eval_ms,
            "timing": "CUDA events recorded inside libffsat on the launching stream (ffsat_eval_profiled, phases "
                      "serialised), mean over the profiled evaluations"}


def reexec_under_torchrun(args):
    """`bench.py --gpus N` outside torchrun: run this same command under torch.distributed.run with N ranks."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ffsat", choices=["ffsat", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--round-len", type=int, default=10)
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tts-seeds", type=int, default=3, help="time-to-solve seeds on the planted c2 instance (0 = skip)")
    ap.add_argument("--tts-cap", type=float, default=10.0, help="per-seed wall-clock cap in seconds (PAR-2 uses 2x)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        reexec_under_torchrun(args)
    rank, world, local = env_rank()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    cfg = CONFIGS[args.config]

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cfg, cfg["make"]())
        return

    import torch
    import torch.distributed as dist
    import paper_2308_15020_b200 as P
    from paper_2308_15020_b200 import dist as D

    # one GPU per rank over NCCL; with fewer visible GPUs than ranks (a dry run on a 1-GPU box) the ranks share the
    # devices over gloo (NCCL refuses two ranks on one device); FFSAT_DIST_BACKEND overrides
    ndev = torch.cuda.device_count()
    backend = os.environ.get("FFSAT_DIST_BACKEND", "nccl" if ndev >= world else "gloo")
    if backend != "nccl":
        local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    inst = cfg["make"]()
    B = cfg["B"]
    if cfg["mode"] == "constraint":
        se = D.ShardedEval(inst.arrays(), rank, world, device=local, batch_ref=B)
        ctx = se.ctx
    else:
        ctx = P.Context.from_instance(inst, device=local, batch_ref=B)
    info = ctx.info
    L = inst.n_lits                       # literal-gradient terms per point of the whole formula
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    dt = torch.float64 if info["precision"] == 64 else torch.float32

    if cfg["mode"] == "constraint":
        xs = torch.from_numpy(synth.points("U", B, inst.n, 1000, np.float64)).to(dt).to(dev)
        # over several ranks the C3 all-reduce of one half of the batch overlaps the evaluation of the other half
        # (ShardedEval chunks; the same bits as one block); FFSAT_C3_CHUNKS overrides
        c3_chunks = int(os.environ.get("FFSAT_C3_CHUNKS", "2" if world > 1 else "1"))

        def step(i):
            se.eval(xs, chunks=c3_chunks)
    else:
        search = ctx.search(B, seed=20230815, point0=rank * B, max_inner=args.round_len, check_every=args.round_len)
        rs = D.RestartSharded(search, args.round_len, rank, world)
        rs.begin()

        def step(i):
            rs.step(i)

    # prime every code path of a step (round end included: CUDA lazy module loading, the collectives) so the first
    # timed round end does not pay one-time costs; then the W warm-up steps
    for i in range(args.round_len):
        step(i)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launch_count()
    evs = []
    for i in range(args.steps):
        if not args.no_flush:
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(args.warmup + i)
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    launches = ctx.launch_count() - launches0
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = sum(step_ms)
    if os.environ.get("FFSAT_BENCH_DUMP"):
        print("step_ms", " ".join(f"{v:.3f}" for v in step_ms), file=sys.stderr)
    clk = clocks.stop()
    t_local = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_max = float(t_local.item())
    B_total = B * world if cfg["mode"] == "restart" else B
    value = L * B_total * args.steps / (ms_max * 1e-3)

    # ---- e2e: the public API with pinned host buffers (H2D of x, D2H of f and grad every step):
    # ffsat_eval with host pointers (restart mode), or host -> device copy + ShardedEval + device -> host
    xh = torch.from_numpy(synth.points("U", B, inst.n, 1000 + rank, np.float64)).to(dt).pin_memory()
    fh = torch.empty(B, dtype=torch.float64).pin_memory()
    gh = torch.empty((B, inst.n), dtype=dt).pin_memory()
    e2e_steps = max(5, min(args.steps, 50))
    if cfg["mode"] == "constraint":
        def host_eval():
            se.eval_host(xh, fh, gh, chunks=c3_chunks)   # one rank: ffsat_eval's pipelined host staging
    else:
        def host_eval():
            P.ffsat_eval(ctx.ptr, xh, B, fh, gh)   # synchronous: H2D, kernels, D2H
    for _ in range(3):
        host_eval()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_ms = []
    for _ in range(e2e_steps):
        if not args.no_flush:
            flush.zero_()
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        host_eval()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    te = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = L * B_total * e2e_steps / (float(te.item()) * 1e-3)
    esz = 8 if info["precision"] == 64 else 4
    e2e = {"value": e2e_value, "unit": "terms/s", "h2d_bytes_per_step": B * inst.n * esz,
           "d2h_bytes_per_step": B * 8 + B * inst.n * esz}

    # ---- roofline of the dominant kernel: per-phase CUDA events on the launching stream
    xd = torch.from_numpy(synth.points("U", B, inst.n, 1000 + rank, np.float64)).to(dt).to(dev)
    fd = torch.empty(B, dtype=torch.float64, device=dev)
    gd = torch.empty_like(xd)
    ud = torch.empty(B, dtype=torch.int32, device=dev)
    phases = []
    for i in range(max(5, min(args.steps, 50))):
        if not args.no_flush:
            flush.zero_()
        # the evaluation of a PGD iteration between checks (no fused check: 9 of every 10 iterations at round_len 10;
        # bench's check iterations and the ffsat_eval API count unsat as well)
        phases.append(ctx.eval_profiled(xd, fd, gd, None if cfg["mode"] == "restart" else ud))
    ph = np.mean(np.array(phases[2:]), axis=0)  # ms: fast, root, grad-reduce, f-reduce
    roofline = roofline_of(info, inst, B, ph, args)

    tts = None
    if args.config == "c2" and args.tts_seeds > 0 and cfg["mode"] == "restart":
        del search, rs
        tts = time_to_solve(P, D, args, local, rank, world, dist)

    if rank == 0:
        base = None if args.no_cpu_baseline or world > 1 else cpu_baseline(cfg, inst, xd.cpu().numpy())
        line = {"metric": "literal-gradient terms/s", "value": value, "unit": "terms/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak" if cfg["mode"] == "restart" else "strong", "vs_baseline": None,
                "dtype": "f64" if info["precision"] == 64 else "f32", "data": "synthetic",
                "config": {"workload": cfg["desc"], "n": inst.n, "m": inst.m, "literals": L,
                           "batch_per_gpu": B, "global_batch": B_total, "round_len": args.round_len,
                           "parallelism": (f"{cfg['mode']}-sharded x{world} ({backend})" if world > 1 else "single GPU"),
                           "l2": "flushed between timed steps (256 MiB write, untimed)" if not args.no_flush else "not flushed",
                           "path": "tiled" if info["path"] == 1 else "global"},
                "evals_per_s": B_total * args.steps / (ms_max * 1e-3),
                "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "clocks": clk}
        if base is not None:
            line["cpu_baseline"] = base
        if tts is not None:
            line["time_to_solve"] = tts
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
