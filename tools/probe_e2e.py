"""Where does e2e lose time vs the device-timed loop?  Variants of the e2e loop."""
import time, torch
import paper_2406_12080_b200 as hs
from paper_2406_12080_b200 import _native as N, scenes
cfg = scenes.CONFIGS["c2"]
h = scenes.hierarchy(cfg)
r = hs.Renderer(0, exact=True)
dh = r.upload(h, validate=False)
L = N.lib()
cams = [c.to_c() for c in scenes.trajectory(cfg, 45, first=0)]
W, H = cfg.width, cfg.height
f32 = N.C.POINTER(N.C.c_float)
frames = [r._frame] + [N.C.c_void_p() for _ in range(3)]
for f in frames[1:]:
    hs._check(L.hs_frame_create(r.ctx, N.C.byref(f)), r.ctx)
for f in frames:
    hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[0], cfg.tau, r._cut, f, None), r.ctx)
pinned = [torch.empty(5 * W * H, dtype=torch.float32, pin_memory=True) for _ in range(4)]
outs = [(N.C.cast(p.data_ptr(), f32), N.C.cast(p.data_ptr() + 12 * W * H, f32),
         N.C.cast(p.data_ptr() + 16 * W * H, f32)) for p in pinned]
rc = N.C.c_int32()
r.set_async(True)

def run(nf, download, timed):
    r.synchronize(); torch.cuda.synchronize()
    t0 = time.perf_counter(); tenq = 0.0
    for i, c in enumerate(cams[5:]):
        fi = i % nf
        if download and i >= nf:
            hs._check(L.hs_frame_download_wait(r.ctx, frames[fi], N.C.byref(rc)), r.ctx)
        a = time.perf_counter()
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, c, cfg.tau, r._cut, frames[fi], None), r.ctx)
        tenq += time.perf_counter() - a
        if download:
            hs._check(L.hs_frame_download_async(r.ctx, frames[fi], *outs[fi]), r.ctx)
    if download:
        for i in range(max(0, 40 - nf), 40):
            hs._check(L.hs_frame_download_wait(r.ctx, frames[i % nf], N.C.byref(rc)), r.ctx)
    r.synchronize()
    dt = time.perf_counter() - t0
    print(f"frames={nf} download={download}: {40/dt:.1f} fps, enqueue {1e3*tenq/40:.3f} ms/frame")

for nf, d in ((1, False), (2, False), (2, True), (3, True), (4, True), (1, True)):
    run(nf, d, True)
    run(nf, d, True)
