"""Summarise an .ncu-rep (details + stall reasons) for profiles/."""
import csv, subprocess, sys, io
rep = sys.argv[1]
def page(p):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))
rows = page("details")
h = rows[0]
ni, vi, ui, si, ki = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Section Name"), h.index("Kernel Name")
keep = {"Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy", "Executed Ipc Active",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Eligible Warps Per Scheduler",
        "No Eligible", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size", "Waves Per SM"}
cur = None
for r in rows[1:]:
    if r[ki] != cur:
        cur = r[ki]; print("==", cur[:110])
    if r[ni] in keep:
        print(f"   {r[ni]} = {r[vi]} {r[ui]}")
raw = page("raw")
hh = raw[0]
for r in raw[2:]:
    print("== stalls (pc samples):", r[hh.index("Kernel Name")][:60])
    items = []
    for i, k in enumerate(hh):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try: items.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i].replace(",", ""))))
            except ValueError: pass
    tot = sum(v for _, v in items) or 1
    print("   " + ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in sorted(items, key=lambda x: -x[1])[:8]))
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in hh: print(f"   {k} = {r[hh.index(k)]} {raw[1][hh.index(k)]}")
