"""Frame lanes (HS_OPT_LANES): frames rendered on frame objects bound to
different streams overlap on the device; results must be bit-identical to
frame-after-frame rendering, including when one cut object is written and read
from two lanes (the cut's cross-lane hazard tracking)."""
import ctypes as C

import numpy as np
import pytest

import paper_2406_12080_b200 as hs
from paper_2406_12080_b200 import _native as N
from paper_2406_12080_b200 import scenes

pytestmark = pytest.mark.gpu


def _images(L, r, fr, w, h):
    col = np.empty(3 * w * h, np.float32)
    dep = np.empty(w * h, np.float32)
    tr = np.empty(w * h, np.float32)
    rc = C.c_int32()
    f32 = C.POINTER(C.c_float)
    hs._check(L.hs_frame_download(r.ctx, fr, col.ctypes.data_as(f32), dep.ctypes.data_as(f32),
                                  tr.ctypes.data_as(f32), C.byref(rc)), r.ctx)
    return np.concatenate([col, dep, tr]).view(np.uint32), int(rc.value)


def _new(L, r, kind):
    p = C.c_void_p()
    hs._check(getattr(L, f"hs_{kind}_create")(r.ctx, C.byref(p)), r.ctx)
    return p


def test_lanes_bit_exact_and_shared_cut():
    cfg = scenes.CONFIGS["c1"]
    h = scenes.hierarchy(cfg)
    cams = [c.to_c() for c in scenes.trajectory(cfg, 8)]
    w, hh = cfg.width, cfg.height
    L = N.lib()
    r = hs.Renderer(0)
    try:
        dh = r.upload(h, validate=False)
        # frame after frame on the default (lane 0) objects
        ref = []
        for c in cams:
            hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, c, cfg.tau, r._cut, r._frame, None), r.ctx)
            ref.append(_images(L, r, r._frame, w, hh))
        # bench_path's odd frame: the previous cut with the next camera
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[2], cfg.tau, r._cut, r._frame, None), r.ctx)
        hs._check(L.hs_render_cut(r.ctx, dh.handle, r._cut, cams[3], r._frame, None), r.ctx)
        ref_reuse = _images(L, r, r._frame, w, hh)

        r.set_lanes(2)
        fa, fb = _new(L, r, "frame"), _new(L, r, "frame")
        ca, cb = _new(L, r, "cut"), _new(L, r, "cut")
        # synchronous first renders bind fa -> lane 1, fb -> lane 0 and size their buffers
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[0], cfg.tau, ca, fa, None), r.ctx)
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[0], cfg.tau, cb, fb, None), r.ctx)
        r.set_async(True)
        for i in range(0, len(cams), 2):
            hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[i], cfg.tau, ca, fa, None), r.ctx)
            hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[i + 1], cfg.tau, cb, fb, None), r.ctx)
            r.set_async(False)
            ia, ib = _images(L, r, fa, w, hh), _images(L, r, fb, w, hh)
            assert np.array_equal(ia[0], ref[i][0]) and ia[1] == ref[i][1]
            assert np.array_equal(ib[0], ref[i + 1][0]) and ib[1] == ref[i + 1][1]
            r.set_async(True)
        # one cut object across the lanes: written on lane 1 (fa), read on lane 0 (fb),
        # then rewritten on lane 1 while fb may still be reading it
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[2], cfg.tau, ca, fa, None), r.ctx)
        hs._check(L.hs_render_cut(r.ctx, dh.handle, ca, cams[3], fb, None), r.ctx)
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[6], cfg.tau, ca, fa, None), r.ctx)
        r.set_async(False)
        ib, ia = _images(L, r, fb, w, hh), _images(L, r, fa, w, hh)
        assert np.array_equal(ib[0], ref_reuse[0]) and ib[1] == ref_reuse[1]
        assert np.array_equal(ia[0], ref[6][0]) and ia[1] == ref[6][1]
        # the context stream joins both lanes
        hs._check(L.hs_context_join(r.ctx), r.ctx)
        r.synchronize()
        for p in (fa, fb):
            L.hs_frame_destroy(p)
        for p in (ca, cb):
            L.hs_cut_destroy(p)
    finally:
        r.close()


def test_cut_capacity_growth(monkeypatch):
    """A cut larger than a frame object's per-splat buffers is flagged on the device
    (nothing rendered); a synchronous call grows the buffers and re-runs the frame,
    an asynchronous one reports CapacityExceeded at the wait."""
    cfg = scenes.CONFIGS["c1"]
    h = scenes.hierarchy(cfg)
    cams = [c.to_c() for c in scenes.trajectory(cfg, 3)]
    w, hh = cfg.width, cfg.height
    L = N.lib()
    ref = hs.Renderer(0)
    small = None
    try:
        dr = ref.upload(h, validate=False)
        hs._check(L.hs_render_hierarchy(ref.ctx, dr.handle, cams[0], cfg.tau, ref._cut, ref._frame, None), ref.ctx)
        a = _images(L, ref, ref._frame, w, hh)
        # frame objects size their per-splat buffers at their first render
        monkeypatch.setenv("HS_CUT_CAP_INIT", "1000")
        small = hs.Renderer(0)
        ds = small.upload(h, validate=False)
        hs._check(L.hs_render_hierarchy(small.ctx, ds.handle, cams[0], cfg.tau, small._cut, small._frame, None),
                  small.ctx)
        b = _images(L, small, small._frame, w, hh)
        assert np.array_equal(a[0], b[0]) and a[1] == b[1]
        # async on a fresh small object: the wait reports the overflow
        fr, cu = _new(L, small, "frame"), _new(L, small, "cut")
        small.set_async(True)
        hs._check(L.hs_render_hierarchy(small.ctx, ds.handle, cams[1], cfg.tau, cu, fr, None), small.ctx)
        assert L.hs_frame_wait(small.ctx, fr) == 103  # HS_CAPACITY_EXCEEDED
        small.set_async(False)
        L.hs_frame_destroy(fr)
        L.hs_cut_destroy(cu)
    finally:
        if small is not None:
            small.close()
        ref.close()


def test_lanes_random_schedule():
    """Random mix of render_hierarchy / render_cut calls over shared cut objects and
    frame objects bound to three lanes, all asynchronous: every frame object's final
    image equals a frame-after-frame replay of its last call."""
    cfg = scenes.CONFIGS["c1"]
    h = scenes.hierarchy(cfg)
    cams = [c.to_c() for c in scenes.trajectory(cfg, 6)]
    w, hh = cfg.width, cfg.height
    L = N.lib()
    rng = np.random.default_rng(7)
    r = hs.Renderer(0)
    ref = hs.Renderer(0)
    try:
        dh = r.upload(h, validate=False)
        dref = ref.upload(h, validate=False)
        r.set_lanes(3)
        frames = [_new(L, r, "frame") for _ in range(3)]
        cuts = [_new(L, r, "cut") for _ in range(2)]
        for f in frames:  # bind lanes, size buffers
            hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[0], cfg.tau, cuts[0], f, None), r.ctx)
        cut_cam = [0, None]  # camera each cut object was selected for
        hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[1], cfg.tau, cuts[1], frames[0], None), r.ctx)
        cut_cam[1] = 1
        last = {}  # frame index -> (cut camera, render camera)
        r.set_async(True)
        for _ in range(24):
            fi, ci, cam = int(rng.integers(3)), int(rng.integers(2)), int(rng.integers(len(cams)))
            if rng.random() < 0.5:
                hs._check(L.hs_render_hierarchy(r.ctx, dh.handle, cams[cam], cfg.tau, cuts[ci], frames[fi], None),
                          r.ctx)
                cut_cam[ci] = cam
                last[fi] = (cam, cam)
            else:
                hs._check(L.hs_render_cut(r.ctx, dh.handle, cuts[ci], cams[cam], frames[fi], None), r.ctx)
                last[fi] = (cut_cam[ci], cam)
        r.set_async(False)
        for fi, (cc, rc) in last.items():
            got = _images(L, r, frames[fi], w, hh)
            hs._check(L.hs_render_hierarchy(ref.ctx, dref.handle, cams[cc], cfg.tau, ref._cut, ref._frame, None),
                      ref.ctx)
            if rc != cc:
                hs._check(L.hs_render_cut(ref.ctx, dref.handle, ref._cut, cams[rc], ref._frame, None), ref.ctx)
            want = _images(L, ref, ref._frame, w, hh)
            assert np.array_equal(got[0], want[0]) and got[1] == want[1], (fi, cc, rc)
        for p in frames:
            L.hs_frame_destroy(p)
        for p in cuts:
            L.hs_cut_destroy(p)
    finally:
        r.close()
        ref.close()
