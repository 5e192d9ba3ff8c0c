"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum]
--csv): launches, mean and total us, mean DRAM bytes per launch.  With a second argument "<config>" the per-launch DRAM
bytes are merged into profiles/ncu_summary.json as "<config>:<kernel base name>" (bench.py's roofline.traffic)."""
import collections
import csv
import json
import os
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
idi = hdr.index("ID")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3, "ms": 1e3}
t = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    if len(r) <= vi:
        continue
    names[r[idi]] = r[ki].split("(")[0].replace("void ", "").replace("ffsat::dev::", "").replace("ffsat::", "")
    t[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in t.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print("kernel,launches,total_us,mean_us,share,mean_dram_bytes")
for name, (n, us, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name},{n},{us:.1f},{us / n:.2f},{us / tot:.3f},{by / n:.0f}")
if len(sys.argv) > 2:
    cfg = sys.argv[2]
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_summary.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    # kernels of this config that the new launch list no longer shows (a changed plan) are dropped
    bases = {name.split("<")[0] for name in agg}
    for key in [k for k in d if k.startswith(f"{cfg}:") and k.split(":", 1)[1] not in bases]:
        del d[key]
    for name, (n, us, by) in agg.items():
        base = name.split("<")[0]
        if base.startswith("at::") or "Functor" in name:
            continue
        key = f"{cfg}:{base}"
        e = d.get(key, {})
        # several instantiations of one kernel: keep the one launched most
        if e.get("launches", 0) <= n:
            d[key] = dict(e, dram_bytes_per_launch=by / n, duration_us_ncu=us / n, launches=n, source="ncu launch list")
    json.dump(d, open(p, "w"), indent=1)
