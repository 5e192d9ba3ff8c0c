"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv): launches, mean and total us."""
import csv, collections, sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.defaultdict(list)
for r in rows[1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0].replace("void ", "").replace("ffsat::dev::", "")
        tot[name].append(float(r[vi].replace(",", "")) / 1e3)
for name, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
    print(f"{name[:60]:60s} n={len(v):4d} mean={sum(v) / len(v):9.2f} us total={sum(v):10.1f} us")
