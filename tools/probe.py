"""Quick perf probe: C2 frames timed with CUDA events on the context stream."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_12080_b200 as hs
from paper_2406_12080_b200 import scenes
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = scenes.CONFIGS[cfgname]
t = time.time(); h = scenes.hierarchy(cfg); print("synth", time.time() - t, flush=True)
r = hs.Renderer(0, exact=True)
t = time.time(); dh = r.upload(h, validate=False); print("upload", time.time() - t, flush=True)
cams = scenes.trajectory(cfg, 20, first=100)
st = hs.StageTimes()
for i, cam in enumerate(cams[:3]):
    out = r.render_hierarchy(dh, cam, cfg.tau, stages=st)
    print("frame", i, out.info, "rc", out.rendered_count, "T mean", float(out.transmittance.mean()), flush=True)
print("stages (3 frames, ms)", {k: round(v * 1e3 / 3, 3) for k, v in vars(st).items()})
for mode in (0, 1):
    r.set_exact(mode == 0)
    stream = torch.cuda.ExternalStream(r.stream_handle())
    r.set_async(True)
    for cam in cams[:3]:
        hs._native.lib().hs_render_hierarchy(r.ctx, dh.handle, cam.to_c(), cfg.tau, r._cut, r._frame, None)
        hs._native.lib().hs_frame_wait(r.ctx, r._frame)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for cam in cams:
        hs._native.lib().hs_render_hierarchy(r.ctx, dh.handle, cam.to_c(), cfg.tau, r._cut, r._frame, None)
    e1.record(stream)
    torch.cuda.synchronize(); r.synchronize()
    st = hs._native.lib().hs_frame_wait(r.ctx, r._frame)
    ms = e0.elapsed_time(e1) / len(cams)
    print("mode", "exact" if mode == 0 else "fast", "ms/frame", ms, "fps", 1000 / ms, "status", st, flush=True)
    r.set_async(False)
