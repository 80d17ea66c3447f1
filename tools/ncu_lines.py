"""Per-source-line instruction and stall-sample shares of one kernel in an .ncu-rep
(ncu --page source --print-source cuda,sass).  Usage: ncu_lines.py REP KERNEL_REGEX [FILE_FILTER]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
data, fname = [], ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 8 and r[0].isdigit():
        try:
            data.append((fname, int(r[0]), r[1], float(r[7] or 0), float(r[4] or 0)))
        except ValueError:
            pass
agg = {}
for f, ln, src, ins, smp in data:  # several launches of the kernel: sum per source line
    a = agg.setdefault((f, ln), [f, ln, src, 0.0, 0.0])
    a[3] += ins
    a[4] += smp
data = sorted(agg.values(), key=lambda a: (a[0], a[1]))
ti = sum(d[3] for d in data) or 1
ts = sum(d[4] for d in data) or 1
print(f"total warp instructions {ti:.4g}")
for f, ln, src, ins, smp in data:
    if ins / ti > 0.004 or smp / ts > 0.01:
        print(f"{f[:12]:12s}{ln:5d} {100*ins/ti:5.1f}% ins {100*smp/ts:5.1f}% smp  {src.strip()[:90]}")
