"""Per-kernel times of one frame from an ncu --metrics gpu__time_duration.sum CSV."""
import csv, sys
lines = open(sys.argv[1]).read().splitlines()
i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[i:]))
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
data = [(r[ki].split("(")[0].replace("void ", "")[:40], float(r[vi].replace(",", ""))) for r in rows[1:] if len(r) > vi]
starts = [j for j, (k, v) in enumerate(data) if "k_select_cut" in k]
fr = int(sys.argv[2]) if len(sys.argv) > 2 else len(starts) - 2
s, e = starts[fr], starts[fr + 1]
tot = sum(v for _, v in data[s:e])
for k, v in data[s:e]:
    print(f"{k:42s} {v / 1000:8.1f} us  {100 * v / tot:5.1f}%")
print(f"{'sum':42s} {tot / 1000:8.1f} us")
