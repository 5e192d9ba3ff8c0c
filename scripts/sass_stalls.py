"""Stall-reason totals and the hottest instruction regions of an ncu --page source --print-source sass CSV export."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr)]
iS, iW, iE = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for r in data:
    for h in reasons:
        tot[h] += int(r[hdr.index(h)] or 0)
T = sum(tot.values())
print("samples", T)
for h, v in tot.most_common(10): print(f"  {h:24s} {v / T * 100:5.1f}%")
W = int(sys.argv[2]) if len(sys.argv) > 2 else 60
print(f"regions of {W} instructions with >= 2% of the samples (top reasons):")
for a in range(0, len(data), W):
    seg = data[a:a + W]
    s = sum(int(r[iW] or 0) for r in seg)
    if s < 0.02 * T: continue
    c = collections.Counter()
    for r in seg:
        for h in reasons: c[h] += int(r[hdr.index(h)] or 0)
    top = ", ".join(f"{h[6:]} {v / s * 100:.0f}%" for h, v in c.most_common(3))
    ops = collections.Counter(r[iS].split()[0] if not r[iS].strip().startswith("@") else r[iS].split()[1] for r in seg)
    print(f"{a:5d} {s / T * 100:5.1f}%  [{top}]  ops: {dict(ops.most_common(4))}")
