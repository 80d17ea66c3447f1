"""Per-task blend timing (a libhsplat_b200.so built with -DHS_BLEND_PROF=1): where the
blend's time goes across its (tile, block) tasks -- the kernel span, the longest tasks
and when they started, and the idle SM time at the end.  Run under gpurun:
  python tools/blend_tasks.py [frame ...]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2406_12080_b200 as hs
from paper_2406_12080_b200 import _native as N
from paper_2406_12080_b200 import scenes

cfg = scenes.CONFIGS[os.environ.get("CFG", "c2")]
frames = [int(a) for a in sys.argv[1:]] or [100]
r = hs.Renderer(0, exact=True)
h = scenes.hierarchy(cfg)
dh = r.upload(h)
L = N.lib()
L.hs_debug_blend_prof.argtypes = [C.POINTER(C.c_ulonglong), C.c_ulonglong]
for f in frames:
    cam = scenes.camera(cfg, f)
    for _ in range(3):
        r.render_hierarchy(dh, cam, cfg.tau)
    ts = r.frame_debug()["tile_start"].astype(np.int64)
    tiles = len(ts) - 1
    tasks = tiles * 8
    buf = np.zeros(3 * tasks, np.uint64)
    assert L.hs_debug_blend_prof(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), tasks) == 0
    t0, t1, meta = buf[0::3].astype(np.int64), buf[1::3].astype(np.int64), buf[2::3]
    sm = (meta >> np.uint64(32)).astype(np.int64)
    batches = (meta & np.uint64(0xFFFFFFFF)).astype(np.int64)
    base = t0.min()
    s, e = (t0 - base) / 1e3, (t1 - base) / 1e3
    d = e - s
    span = e.max()
    n_tile = np.diff(ts)
    print(f"frame {f}: tasks {tasks} span {span:.1f} us, sum of task time {d.sum():.0f} us, "
          f"mean {d.mean():.2f} us, last task start {s.max():.1f} us")
    # per-SM busy end: when each SM's last task ended
    ends = np.zeros(sm.max() + 1)
    np.maximum.at(ends, sm, e)
    print(f"  SM last-task end: min {ends.min():.1f} median {np.median(ends):.1f} max {ends.max():.1f} us")
    order = np.argsort(-d)[:15]
    for i in order:
        print(f"  task {i:6d} (rank tile {i >> 3}, blk {i & 7}) start {s[i]:7.1f} end {e[i]:7.1f} dur {d[i]:7.1f} us "
              f"batches {batches[i]:5d} sm {sm[i]}")
    for q in (50, 90, 99, 99.9):
        print(f"  task duration p{q}: {np.percentile(d, q):.1f} us")
