"""Per-tile list lengths of C2 frames (the in-tile sort's size classes): run under gpurun."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_12080_b200 as hs
from paper_2406_12080_b200 import scenes

cfg = scenes.CONFIGS["c2"]
r = hs.Renderer(0, exact=True)
h = scenes.hierarchy(cfg)
dh = r.upload(h)
for f in (0, 100, 500):
    out = r.render_hierarchy(dh, scenes.camera(cfg, f), cfg.tau)
    ts = r.frame_debug()["tile_start"].astype(np.int64)
    n = np.diff(ts)
    D = int(n.sum())
    print(f"frame {f}: tiles {len(n)} D {D} mean {n.mean():.0f} max {n.max()}")
    for lo, hi in ((0, 1), (1, 512), (512, 1024), (1024, 2048), (2048, 4096), (4096, 1 << 40)):
        m = (n >= lo) & (n < hi)
        print(f"  [{lo},{hi}) tiles {int(m.sum()):6d} entries {int(n[m].sum()):9d} ({100 * n[m].sum() / D:5.1f}%)")
