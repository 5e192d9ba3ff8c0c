"""Copy this round's GPU evidence into profiles/: ncu launch lists, per-kernel --set full summaries, the
dram bytes per launch bench.py reports as roofline.traffic, and the bench lines."""
import csv, io, json, os, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, PR = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(PR, exist_ok=True)
summ_path = os.path.join(PR, "ncu_summary.json")
summary = json.load(open(summ_path)) if os.path.exists(summ_path) else {}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return {h: v for h, v in zip(r[0], r[2])}, {h: u for h, u in zip(r[0], r[1])}


def num(v):
    return float(str(v).replace(",", ""))


for rep, cfg, kname in (("prof_tmem", "c2", "fast_tmem_kernel"), ("prof_tmem_chk", "c2", "fast_tmem_kernel_check"),
                        ("prof_tiled", "c2", "fast_wide_kernel"), ("prof_sym", "c3", "sym_item_kernel"),
                        ("prof_tree", "c3", "sym_tree_kernel"), ("prof_own", "c5", "owner_grp_kernel"),
                        ("prof_global", "c5", "fast_global_kernel"), ("prof_short", "c4", "fast_global_kernel"),
                        ("prof_long", "c4", "fast_global_long_kernel"), ("prof_reduce5", "c5", "reduce_grad_kernel")):
    p = os.path.join(G, rep + ".ncu-rep")
    if not os.path.exists(p):
        continue
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), p], capture_output=True, text=True).stdout
    with open(os.path.join(PR, f"{tag}_ncu_{cfg}_{kname}.txt"), "w") as fh:
        fh.write(f"# ncu --set full --clock-control none, one launch of {kname} ({rep}.ncu-rep)\n" + txt)
    v, u = raw(p)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    dram = num(v["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]] + \
        num(v["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
    dur = num(v["gpu__time_duration.sum"]) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[u["gpu__time_duration.sum"]]
    summary[f"{cfg}:{kname}"] = {"dram_bytes_per_launch": dram, "duration_us_ncu": dur, "round": tag,
                      "grid": v.get("launch__grid_size"), "block": v.get("launch__block_size"),
                      "registers": v.get("launch__registers_per_thread"),
                      "fp64_pipe_pct": v.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                      "issue_active_pct": v.get("sm__inst_issued.avg.pct_of_peak_sustained_active")}
json.dump(summary, open(summ_path, "w"), indent=1)


def launches(src, dst):
    p = os.path.join(G, src)
    if not os.path.exists(p):
        return
    rows = list(csv.reader(open(p)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    agg = {}
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += num(d["Metric Value"]) * (1e-3 if d["Metric Unit"] in ("nsecond", "ns") else 1e3 if d["Metric Unit"] in ("msecond", "ms") else 1.0)
    tot = sum(t for _, t in agg.values())
    with open(os.path.join(PR, dst), "w") as fh:
        fh.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)\n")
        fh.write("kernel,launches,total_us,mean_us,share\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"{k},{n},{t:.1f},{t / n:.2f},{t / tot:.3f}\n")


for c in ("c2", "c3", "c4", "c5"):   # per-kernel launch summaries written by scripts/gpu_launches.sh (time + DRAM bytes)
    src = os.path.join(G, f"launch_summary_{c}.csv")
    if os.path.exists(src):
        with open(os.path.join(PR, f"{tag}_launches_{c}.csv"), "w") as fh:
            fh.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                     "(cold-cache, serialised launches; bench.py --config " + c + " --steps 20 --warmup 3)\n")
            fh.write(open(src).read())
for f in sorted(os.listdir(G)):
    if (f.startswith("bench") or f in ("table2_portfolio.json", "rq1_suite.json")) and f.endswith(".json") and \
            os.path.getsize(os.path.join(G, f)):
        shutil.copy(os.path.join(G, f), os.path.join(PR, f"{tag}_{f}"))
print(json.dumps(summary, indent=1))
