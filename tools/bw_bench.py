"""Backward timing on the C2 frame (CUDA events around hs_render_backward's kernels are
not separated from the host copies here; reports the call's wall time and the device
kernel time from ncu separately).  Diagnostic."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_12080_b200 as hs
from paper_2406_12080_b200 import scenes
cfg = scenes.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
h = scenes.hierarchy(cfg)
r = hs.Renderer(0)
dh = r.upload(h, validate=False)
cam = scenes.camera(cfg, 100)
out = r.render_hierarchy(dh, cam, cfg.tau)
lg = np.random.default_rng(1).uniform(-1, 1, (3, cam.height, cam.width)).astype(np.float32)
for rep in range(3):
    t0 = time.perf_counter()
    g = r.render_backward(lg)
    print(f"backward call {1e3 * (time.perf_counter() - t0):.2f} ms, splats {g['mean'].shape[0]}, "
          f"|dmean| {float(np.abs(g['mean']).max()):.3g}")
