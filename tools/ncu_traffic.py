"""Per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum, bytes per
launch, averaged over the captured launches of each kernel) from an ncu --set
full report -> JSON consumed by bench.py's roofline.traffic.
Usage: ncu_traffic.py REP OUT.json"""
import csv, io, json, subprocess, sys
from collections import defaultdict
rep, out = sys.argv[1], sys.argv[2]
PCT = ["smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      ",".join(["dram__bytes_read.sum", "dram__bytes_write.sum"] + PCT)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
ki = h.index("Kernel Name")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
acc = defaultdict(lambda: [0.0, 0.0, 0.0, 0])
pct = defaultdict(lambda: defaultdict(float))
for r in rows[2:]:
    name = r[ki].split("(")[0].replace("void ", "")
    a = acc[name]
    for j, key in enumerate(("dram__bytes_read.sum", "dram__bytes_write.sum")):
        i = h.index(key)
        a[j] += float(r[i].replace(",", "")) * scale.get(units[i], 1)
    a[3] += 1
    for key in PCT:
        if key in h:
            try:
                pct[name][key] += float(r[h.index(key)].replace(",", ""))
            except ValueError:
                pass
res = {"source": rep.split("/")[-1], "how": "ncu --set full --clock-control none, one C2 frame; per-launch mean",
       "kernels": {k: {"dram_bytes": (v[0] + v[1]) / v[3], "read": v[0] / v[3], "write": v[1] / v[3],
                       "launches": v[3],
                       "pct_of_peak": {m.split(".")[0].replace("sm__inst_executed_", "").replace("smsp__", "").replace("gpu__", "")
                                       .replace("__", "_"): pct[k][m] / v[3] for m in PCT}}
                   for k, v in acc.items()}}
json.dump(res, open(out, "w"), indent=1)
for k, v in res["kernels"].items():
    print(f"{k:28s} {v['dram_bytes'] / 1e6:10.2f} MB  x{v['launches']}")
