"""A few C2 in-scene trajectory frames (screen-covering splats), for ncu launch lists:
    python tools/inscene_frames.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_12080_b200 as hs  # noqa: E402
from paper_2406_12080_b200 import scenes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = scenes.CONFIGS["c2"]
h = scenes.hierarchy(cfg)
r = hs.Renderer(0)
dh = r.upload(h, validate=False)
for cam in scenes.trajectory_inscene(cfg, n):
    out = r.render_hierarchy(dh, cam, cfg.tau)
print("inscene frames", n, "last rendered", out.rendered_count, out.info.get("n_duplicates"))
