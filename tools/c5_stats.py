"""Where the C5 (100M-leaf multi-chunk, 4K) duplicates come from: per-splat tile
counts of one frame grouped by what the splat is (skybox vs city, leaf vs
interior, transition or not).  Diagnostic; run under gpurun."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_12080_b200 as hs
from paper_2406_12080_b200 import scenes

cfg = scenes.CONFIGS["c5"]
leaves = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.leaves
r = hs.Renderer(0, exact=True, debug=True)
dh = scenes.multichunk(r, leaves)
cam = scenes.camera(cfg, 0)
out, cut = r.render_hierarchy(dh, cam, cfg.tau, return_cut=True)
dbg = r.frame_debug()
pj = dbg["proj16"]
vis = pj[:, 0] == 0
rect = pj[:, 13].view(np.uint32)
tx0 = pj[:, 14].view(np.int32)
ty0 = pj[:, 15].view(np.int32)
radius = pj[:, 12].view(np.int32)
# tiles per splat from the pre-sort duplicate list
cnt = np.bincount(dbg["dup_vals"], minlength=len(pj))
print("C", len(pj), "V", int(vis.sum()), "D", int(cnt.sum()))
z = pj[:, 1]
far = z > 5000.0
t = cut.t
for name, m in (("sky (z>5km)", far), ("city t=1", ~far & (t >= 1.0)), ("city t<1", ~far & (t < 1.0))):
    m = m & vis
    print(f"{name:14s} splats {int(m.sum()):10d}  dups {int(cnt[m].sum()):12d}  mean tiles {cnt[m].mean() if m.any() else 0:8.2f}"
          f"  mean radius {radius[m].mean() if m.any() else 0:8.2f}")
for lo, hi in ((0, 8), (8, 16), (16, 32), (32, 64), (64, 128), (128, 1 << 30)):
    m = vis & (radius >= lo) & (radius < hi)
    print(f"radius [{lo},{hi}) splats {int(m.sum()):10d} dups {int(cnt[m].sum()):12d}")
print("n_eval", out.info.get("n_eval"), "n_contrib", out.info.get("n_contrib"))
