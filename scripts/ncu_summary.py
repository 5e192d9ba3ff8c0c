"""Summarise an ncu --set full report: key SOL / occupancy / stall metrics and the top SASS stall sites."""
import csv, subprocess, sys, collections, io
rep = sys.argv[1]
def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))
rows = page("details")
hdr = rows[0]
iN, iU, iV = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
keep = ["Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "Executed Instructions"]
seen = set()
for r in rows[1:]:
    if len(r) > iV and r[iN] in keep and r[iN] not in seen:
        seen.add(r[iN]); print(f"{r[iN]:40s} {r[iV]:>14s} {r[iU]}")
raw = page("raw")
h, u, v = raw[0], raw[1], raw[2]
for want in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
             "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_shared_st.sum",
             "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"):
    if want in h:
        i = h.index(want); print(f"{want:70s} {v[i]:>16s} {u[i]}")
s = page("source", ["--print-source=sass"])
sh, sd = s[1], s[2:]
iS, iE, iW = sh.index("Source"), sh.index("Instructions Executed"), sh.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iE] or 0) for r in sd if len(r) > iE); ws = sum(int(r[iW] or 0) for r in sd if len(r) > iE)
ops = collections.Counter(); st = collections.Counter()
for r in sd:
    if len(r) <= iE: continue
    t = r[iS].split()
    if not t: continue
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op.split(".")[0]] += int(r[iE] or 0); st[op.split(".")[0]] += int(r[iW] or 0)
print(f"instructions {tot}, stall samples {ws}")
for k, n in ops.most_common(18): print(f"  {k:10s} {n:12d} {100*n/tot:5.1f}%  stall {100*st[k]/max(ws,1):5.1f}%")
print("top stall sites:")
for r in sorted([r for r in sd if len(r) > iE], key=lambda r: -int(r[iW] or 0))[:12]:
    print(f"  {r[iS][:70]:70s} stall={r[iW]:>6s} exec={r[iE]}")
