"""Workload for compute-sanitizer (racecheck / synccheck / memcheck / initcheck).

A small city (20K leaves, 320x240) rendered through every kernel family the
frame path launches: cut + raster on two frame lanes in async mode with one
cut object shared between the lanes (the cross-lane hazard case), a reused cut
(bench_path's odd frame), a splat render, a backward pass, the fast blend
mode, compaction, heavy tiles through every in-tile sort path, and a short
refinement.  Run as

    compute-sanitizer --tool racecheck python tools/sanitize_frames.py

The script itself checks that the lane results equal frame-after-frame results.
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2406_12080_b200 as hs  # noqa: E402
from paper_2406_12080_b200 import _native as N  # noqa: E402
from paper_2406_12080_b200 import scenes  # noqa: E402


def images(L, r, fr, w, h):
    col = np.empty(5 * w * h, np.float32)
    rc = C.c_int32()
    f32 = C.POINTER(C.c_float)
    base = col.ctypes.data
    hs._check(L.hs_frame_download(r.ctx, fr, C.cast(base, f32), C.cast(base + 12 * w * h, f32),
                                  C.cast(base + 16 * w * h, f32), C.byref(rc)), r.ctx)
    return col.view(np.uint32).copy(), int(rc.value)


def new(L, r, kind):
    p = C.c_void_p()
    hs._check(getattr(L, f"hs_{kind}_create")(r.ctx, C.byref(p)), r.ctx)
    return p


def main():
    cfg = scenes.Config("san_20k", 20_000, 320, 240, 160.0, 3.0, altitude=12.0, standoff=8.0, lookahead=40.0)
    h = hs.synth_city(cfg.leaves, seed=3)
    cams = [c.to_c() for c in scenes.trajectory(cfg, 6, 40)]
    w, hh = cfg.width, cfg.height
    L = N.lib()
    r = hs.Renderer(0)
    dh = r.upload(h, validate=False)
    ref = []
    for c in cams:
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, c, cfg.tau, r._cut, r._frame, None), r.ctx)
        ref.append(images(L, r, r._frame, w, hh))
    # odd frame of bench_path: reuse the cut
    hs._check(L.hs_render_cut(r.ctx, dh.handle, r._cut, cams[1], r._frame, None), r.ctx)
    images(L, r, r._frame, w, hh)
    # two lanes, async, a cut shared between lanes
    r.set_lanes(2)
    fa, fb = new(L, r, "frame"), new(L, r, "frame")
    ca, cb = new(L, r, "cut"), new(L, r, "cut")
    hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[0], cfg.tau, ca, fa, None), r.ctx)
    hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[0], cfg.tau, cb, fb, None), r.ctx)
    r.set_async(True)
    for i in range(0, 4, 2):
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[i], cfg.tau, ca, fa, None), r.ctx)
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[i + 1], cfg.tau, cb, fb, None), r.ctx)
    hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[4], cfg.tau, ca, fa, None), r.ctx)
    hs._check(L.hs_render_cut(r.ctx, dh.handle, ca, cams[5], fb, None), r.ctx)
    r.set_async(False)
    hs._check(L.hs_context_join(r.ctx), r.ctx)
    r.synchronize()
    ia = images(L, r, fa, w, hh)
    assert np.array_equal(ia[0], ref[4][0]), "lane result differs"
    for p in (fa, fb):
        L.hs_frame_destroy(p)
    for p in (ca, cb):
        L.hs_cut_destroy(p)
    # splat render + backward
    cut = r.select_cut(dh, scenes.camera(cfg, 40), cfg.tau)
    sp = r.cut_render_splats(dh, cut)
    out = r.render_forward(sp, scenes.camera(cfg, 40), want_context=True)
    g = np.ones((3, hh, w), np.float32) * 0.01
    r.render_backward(g)
    # fast blend mode
    r.set_exact(False)
    r.render_hierarchy(dh, scenes.camera(cfg, 41), cfg.tau)
    r.set_exact(True)
    # compaction on the device
    r.compact(dh, [scenes.camera(cfg, 40)], 3.0)
    # heavy tiles: a big tile split by key range, an oversized equal-depth partition
    # (chunks + merge), the LSD fallbacks (tests/test_gpu_order.py's cases)
    from tests.fixtures import Rng
    from tests.test_gpu_order import tile_cluster
    for n, same in ((12000, False), (9000, True), (3000, True), (400, True)):
        sp2, cam2 = tile_cluster(Rng(1000 + n), n, 5.0, same)
        r.render_forward(sp2, cam2)
    # a short refinement (refine.cu) with a backward per step
    tgt = [np.clip(out.color * 0.9 + 0.05, 0, 1).astype(np.float32)]
    r.refine_hierarchy(dh, [scenes.camera(cfg, 40)], tgt, hs.RefineConfig(steps=2, tau_min=3.0, tau_max=12.0))
    r.close()
    print("sanitize workload ok", out.rendered_count)


if __name__ == "__main__":
    main()
