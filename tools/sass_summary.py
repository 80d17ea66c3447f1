"""Per-kernel counts of the SASS instructions that show which B200 memory paths a
kernel uses (bulk/TMA copies, cp.async, 256-bit loads, mbarrier ops, FP64), from
cuobjdump of the built objects.  Usage: sass_summary.py OBJ..."""
import re, subprocess, sys
from collections import Counter
KEYS = ["UBLKCP", "UTMALDG", "LDGSTS", "LDG.E.ENL2.256", "LDG.E.128", "SYNCS", "REDUX", "MATCH", "VOTE",
        "DFMA", "DMUL", "MUFU", "SHFL"]
for obj in sys.argv[1:]:
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    fn, cnt = None, Counter()
    def flush():
        if fn and any(cnt.values()):
            print(f"{obj.split('/')[-1]:12s} {fn[:60]:60s} " + " ".join(f"{k}={cnt[k]}" for k in KEYS if cnt[k]))
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            flush()
            fn, cnt = m.group(1), Counter()
            continue
        for k in KEYS:
            if re.search(r"\b" + re.escape(k), line):
                cnt[k] += 1
    flush()
