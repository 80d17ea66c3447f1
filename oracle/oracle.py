"""ctypes wrapper of the CPU oracle (oracle/hsplat_oracle.cpp) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module; the product path never does.
Builds oracle/_build/libhsplat_oracle.so on first use (g++ -O3, no -march, as
the reference's CMake Release build).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libhsplat_oracle.so")

f32p = C.POINTER(C.c_float)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class or_camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("w2c", C.c_float * 12)]


class or_nodes(C.Structure):
    _fields_ = [("parent", u32p), ("first_child", u32p), ("child_count", u32p), ("bmin", f32p), ("bmax", f32p),
                ("mean", f32p), ("scale", f32p), ("rot_wxyz", f32p), ("falloff", f32p), ("sh", f32p)]


class or_splats(C.Structure):
    _fields_ = [("mean", f32p), ("scale", f32p), ("rot_wxyz", f32p), ("sh", f32p), ("falloff", f32p),
                ("parent_falloff", f32p), ("t", f32p), ("siblings", i32p)]


class or_refine_config(C.Structure):
    _fields_ = [("tau_min", C.c_float), ("tau_max", C.c_float), ("steps", C.c_int32), ("lr_mean", C.c_float),
                ("lr_scale", C.c_float), ("lr_rotation", C.c_float), ("lr_falloff", C.c_float),
                ("lr_sh", C.c_float), ("rng_seed", C.c_uint64)]


class or_stage_times(C.Structure):
    _fields_ = [("cut_expand", C.c_double), ("weights", C.c_double), ("preprocess", C.c_double),
                ("duplicate", C.c_double), ("tile_ranges", C.c_double), ("alpha_blend", C.c_double)]


_vp = C.c_void_p
_SIGS = {
    "or_last_error": (C.c_char_p, []),
    "or_set_thread_count": (None, [C.c_int]),
    "or_thread_count": (C.c_int, []),
    "or_granularity": (C.c_float, [f32p, f32p, C.POINTER(or_camera)]),
    "or_interp_weight": (C.c_float, [C.c_float, C.c_float, C.c_float]),
    "or_transition_alpha": (C.c_int, [C.c_float, C.c_int, f32p]),
    "or_expf": (C.c_float, [C.c_float]),
    "or_powf": (C.c_float, [C.c_float, C.c_float]),
    "or_validate_camera": (C.c_int, [C.POINTER(or_camera)]),
    "or_hierarchy_create": (_vp, [C.POINTER(or_nodes), C.c_uint64]),
    "or_hierarchy_free": (None, [_vp]),
    "or_hierarchy_leaf_count": (C.c_uint64, [_vp]),
    "or_hierarchy_size": (C.c_uint64, [_vp]),
    "or_hierarchy_export": (None, [_vp, u32p, u32p, u32p, f32p, f32p, f32p, f32p, f32p, f32p, f32p]),
    "or_render_backward": (C.c_int, [_vp, C.POINTER(or_splats), C.c_uint64, C.POINTER(or_camera), f32p, f32p, f32p,
                                     f32p, f32p, f32p, f32p, f32p, f32p, f32p, f32p, f32p]),
    "or_compact": (C.c_int, [_vp, C.POINTER(or_camera), C.c_uint64, C.c_float, C.c_float, C.POINTER(_vp)]),
    "or_select_cut": (C.c_int, [_vp, C.POINTER(or_camera), C.c_float, u32p, f32p, f32p, u64p, f64p]),
    "or_cut_render_splats": (C.c_int, [_vp, u32p, f32p, f32p, C.c_uint64, f32p, f32p, f32p, f32p, f32p, f32p,
                                       f32p, i32p]),
    "or_frame_new": (_vp, []),
    "or_frame_free": (None, [_vp]),
    "or_render_forward": (C.c_int, [C.POINTER(or_splats), C.c_uint64, C.POINTER(or_camera), _vp, C.c_int]),
    "or_render_reference": (C.c_int, [C.POINTER(or_splats), C.c_uint64, C.POINTER(or_camera), _vp]),
    "or_render_hierarchy": (C.c_int, [_vp, C.POINTER(or_camera), C.c_float, _vp, C.c_int]),
    "or_frame_sizes": (None, [_vp, u64p]),
    "or_frame_images": (None, [_vp, f32p, f32p, f32p]),
    "or_frame_ctx": (None, [_vp, u64p, u32p, u32p, f32p]),
    "or_frame_cut": (None, [_vp, u32p, f32p, f32p]),
    "or_frame_times": (None, [_vp, C.POINTER(or_stage_times)]),
    "or_project": (C.c_int, [C.POINTER(or_splats), C.POINTER(or_camera), f32p, f32p, f32p]),
    "or_bench_path": (C.c_int, [_vp, C.POINTER(or_camera), C.c_uint64, f64p, C.c_uint64, C.c_float, f64p]),
    "or_psnr": (C.c_double, [f32p, f32p, C.c_uint64]),
    "or_refine_hierarchy": (C.c_int, [_vp, C.POINTER(or_camera), C.c_uint32, C.POINTER(f32p), f32p,
                                      C.POINTER(or_refine_config), C.POINTER(_vp), f64p, f32p]),
    "or_photometric_loss": (C.c_float, [f32p, f32p, C.c_int32, C.c_int32, f32p]),
}

_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "hsplat_oracle.cpp")
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
            build()
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


def _chk(st):
    if st:
        raise OracleError(st, lib().or_last_error().decode())


def _p(a, ct):
    if a is None:
        return C.cast(None, C.POINTER(ct))
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ct))


def camera(cam) -> or_camera:
    c = or_camera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    w = np.ascontiguousarray(cam.world_to_camera, np.float32).reshape(12)
    for i in range(12):
        c.w2c[i] = float(w[i])
    return c


def set_thread_count(n: int):
    lib().or_set_thread_count(int(n))


def thread_count() -> int:
    return int(lib().or_thread_count())


class OracleHierarchy:
    """The reference's AoS Hierarchy (std::vector<HierarchyNode>) built from host SoA arrays."""

    def __init__(self, h):
        h = h.contiguous()
        self._keep = h
        s = or_nodes()
        s.parent, s.first_child, s.child_count = (_p(h.parent, C.c_uint32), _p(h.first_child, C.c_uint32),
                                                  _p(h.child_count, C.c_uint32))
        s.bmin, s.bmax, s.mean, s.scale = (_p(h.bmin, C.c_float), _p(h.bmax, C.c_float), _p(h.mean, C.c_float),
                                           _p(h.scale, C.c_float))
        s.rot_wxyz, s.falloff, s.sh = _p(h.rot_wxyz, C.c_float), _p(h.falloff, C.c_float), _p(h.sh, C.c_float)
        self.n = h.n
        self.handle = lib().or_hierarchy_create(C.byref(s), h.n)

    def leaf_count(self) -> int:
        return int(lib().or_hierarchy_leaf_count(self.handle))

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.or_hierarchy_free(self.handle)
            self.handle = None


def select_cut(oh: OracleHierarchy, cam, tau: float):
    n = oh.n
    node = np.empty(n, np.uint32)
    t = np.empty(n, np.float32)
    a = np.empty(n, np.float32)
    cnt = C.c_uint64()
    sec = C.c_double()
    _chk(lib().or_select_cut(oh.handle, C.byref(camera(cam)), float(tau), _p(node, C.c_uint32), _p(t, C.c_float),
                             _p(a, C.c_float), C.byref(cnt), C.byref(sec)))
    k = cnt.value
    return node[:k].copy(), t[:k].copy(), a[:k].copy()


def cut_render_splats(oh: OracleHierarchy, node, t, alpha=None):
    from paper_2406_12080_b200 import RenderSplats  # container type only
    n = len(node)
    out = RenderSplats.empty(n)
    node = np.ascontiguousarray(node, np.uint32)
    t = np.ascontiguousarray(t, np.float32)
    alpha = None if alpha is None else np.ascontiguousarray(alpha, np.float32)
    _chk(lib().or_cut_render_splats(oh.handle, _p(node, C.c_uint32), _p(t, C.c_float), _p(alpha, C.c_float), n,
                                    _p(out.mean, C.c_float), _p(out.scale, C.c_float), _p(out.rot_wxyz, C.c_float),
                                    _p(out.sh, C.c_float), _p(out.falloff, C.c_float),
                                    _p(out.parent_falloff, C.c_float), _p(out.t, C.c_float),
                                    _p(out.siblings, C.c_int32)))
    return out


def _splats(sp):
    sp = sp.contiguous()
    s = or_splats()
    s.mean, s.scale, s.rot_wxyz, s.sh = (_p(sp.mean, C.c_float), _p(sp.scale, C.c_float), _p(sp.rot_wxyz, C.c_float),
                                         _p(sp.sh, C.c_float))
    s.falloff, s.parent_falloff, s.t = (_p(sp.falloff, C.c_float), _p(sp.parent_falloff, C.c_float),
                                        _p(sp.t, C.c_float))
    s.siblings = _p(sp.siblings, C.c_int32)
    return s, sp


class OracleFrame:
    def __init__(self):
        self.h = lib().or_frame_new()

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_frame_free(self.h)
            self.h = None

    def sizes(self):
        sz = np.zeros(9, np.uint64)
        lib().or_frame_sizes(self.h, _p(sz, C.c_uint64))
        keys = ["width", "height", "tiles_x", "tiles_y", "n_projected", "n_order", "n_entries", "rendered_count",
                "ncut"]
        return {k: int(v) for k, v in zip(keys, sz)}

    def images(self):
        s = self.sizes()
        H, W = s["height"], s["width"]
        color = np.empty((3, H, W), np.float32)
        depth = np.empty((H, W), np.float32)
        trans = np.empty((H, W), np.float32)
        lib().or_frame_images(self.h, _p(color, C.c_float), _p(depth, C.c_float), _p(trans, C.c_float))
        return color, depth, trans, s["rendered_count"]

    def context(self):
        """ForwardContext (render.hpp:87-98): tile_start, tile_entries, order, per-splat projection dump."""
        s = self.sizes()
        ts = np.empty(s["tiles_x"] * s["tiles_y"] + 1, np.uint64)
        te = np.empty(s["n_entries"], np.uint32)
        order = np.empty(s["n_order"], np.uint32)
        pj = np.empty((s["n_projected"], 16), np.float32)
        lib().or_frame_ctx(self.h, _p(ts, C.c_uint64), _p(te, C.c_uint32), _p(order, C.c_uint32), _p(pj, C.c_float))
        return dict(tile_start=ts, tile_entries=te, order=order, proj16=pj, tiles_x=s["tiles_x"])

    def cut(self):
        n = self.sizes()["ncut"]
        node = np.empty(n, np.uint32)
        t = np.empty(n, np.float32)
        a = np.empty(n, np.float32)
        lib().or_frame_cut(self.h, _p(node, C.c_uint32), _p(t, C.c_float), _p(a, C.c_float))
        return node, t, a

    def times(self):
        st = or_stage_times()
        lib().or_frame_times(self.h, C.byref(st))
        return {k: getattr(st, k) for k, _ in or_stage_times._fields_}


def render_forward(splats, cam, keep_ctx=True) -> OracleFrame:
    s, keep = _splats(splats)
    f = OracleFrame()
    _chk(lib().or_render_forward(C.byref(s), len(keep), C.byref(camera(cam)), f.h, 1 if keep_ctx else 0))
    return f


def render_reference(splats, cam) -> OracleFrame:
    s, keep = _splats(splats)
    f = OracleFrame()
    _chk(lib().or_render_reference(C.byref(s), len(keep), C.byref(camera(cam)), f.h))
    return f


def render_hierarchy(oh: OracleHierarchy, cam, tau: float, keep_ctx=True) -> OracleFrame:
    f = OracleFrame()
    _chk(lib().or_render_hierarchy(oh.handle, C.byref(camera(cam)), float(tau), f.h, 1 if keep_ctx else 0))
    return f


def project(splats, cam):
    """project() of the first splat -> (proj16, cov2d[4], (det_pre, det_post))."""
    s, keep = _splats(splats)
    o = np.empty(16, np.float32)
    cov = np.empty(4, np.float32)
    dets = np.empty(2, np.float32)
    _chk(lib().or_project(C.byref(s), C.byref(camera(cam)), _p(o, C.c_float), _p(cov, C.c_float),
                          _p(dets, C.c_float)))
    return o, cov, dets


def granularity(bmin, bmax, cam) -> float:
    bmin = np.ascontiguousarray(bmin, np.float32)
    bmax = np.ascontiguousarray(bmax, np.float32)
    return float(lib().or_granularity(_p(bmin, C.c_float), _p(bmax, C.c_float), C.byref(camera(cam))))


def interp_weight(en, ep, tau) -> float:
    return float(lib().or_interp_weight(en, ep, tau))


def transition_alpha(a, k) -> float:
    out = C.c_float()
    _chk(lib().or_transition_alpha(float(a), int(k), C.byref(out)))
    return float(out.value)


def bench_path(oh: OracleHierarchy, cams, tau: float) -> np.ndarray:
    arr = (or_camera * len(cams))(*[camera(c) for c in cams])
    stats = np.zeros((len(cams), 9), np.float64)
    _chk(lib().or_bench_path(oh.handle, arr, len(cams), None, 0, float(tau), _p(stats, C.c_double)))
    return stats


def expf(x: float) -> float:
    return float(lib().or_expf(x))


def powf(x: float, y: float) -> float:
    return float(lib().or_powf(x, y))


def consolidate_bfs(parts, root=None):
    """consolidate's breadth-first serialisation (scene.hpp:281-316) of a forest
    in numpy, for forests without cross-chunk pruning.  `parts` are host
    Hierarchy objects (root 0, children contiguous); `root` is None for a single
    part, else a dict with the merged root's fields (mean, scale, rot_wxyz,
    falloff, sh, bmin, bmax) and the re-matched forest roots' `kid_scale` and
    `kid_rot` (k x 3, k x 4).  Returns a dict of SoA arrays in the serialised
    order: children contiguous, parent index < child index."""
    k = len(parts)
    fields = ("bmin", "bmax", "mean", "scale", "rot_wxyz", "falloff", "sh")
    off = 1 if k > 1 else 0  # the merged global root takes index 0
    # BFS level by level: a level is, in order, every previous-level node's child range
    level = [(p, np.zeros(1, np.int64), np.full(1, 0 if k > 1 else 0xFFFFFFFF, np.int64)) for p in range(k)]
    order_p, order_j, order_par = [], [], []
    pos = off
    while level:
        nxt = []
        for p, j, par in level:
            h = parts[p]
            order_p.append(np.full(len(j), p)), order_j.append(j), order_par.append(par)
            cc = h.child_count[j].astype(np.int64)
            fc = h.first_child[j].astype(np.int64)
            kids = np.repeat(fc, cc) + (np.arange(cc.sum()) - np.repeat(np.cumsum(cc) - cc, cc))
            if len(kids):
                nxt.append((p, kids, np.repeat(pos + np.arange(len(j)), cc)))
            pos += len(j)
        level = nxt
    P, J, PAR = np.concatenate(order_p), np.concatenate(order_j), np.concatenate(order_par)
    n = len(P) + off
    out = {f: np.zeros((n,) + getattr(parts[0], f).shape[1:], np.float32) for f in fields}
    out["parent"] = np.zeros(n, np.uint32)
    out["child_count"] = np.zeros(n, np.uint32)
    for p in range(k):
        sel = np.flatnonzero(P == p)
        for f in fields:
            out[f][off + sel] = getattr(parts[p], f)[J[sel]]
        out["child_count"][off + sel] = parts[p].child_count[J[sel]]
    out["parent"][off:] = PAR.astype(np.uint32)
    if k > 1:
        for f in fields:
            out[f][0] = root[f]
        out["parent"][0] = 0xFFFFFFFF
        out["child_count"][0] = k
        out["scale"][1:1 + k] = root["kid_scale"]
        out["rot_wxyz"][1:1 + k] = root["kid_rot"]
    # children of node i start after the root and all earlier nodes' children
    cc = out["child_count"].astype(np.int64)
    first = 1 + np.cumsum(cc) - cc
    out["first_child"] = np.where(cc > 0, first, 0xFFFFFFFF).astype(np.uint32)
    return out


def compact(oh: OracleHierarchy, cams, tau_min: float = 3.0, tau_max: float = 0.0) -> dict:
    """compact (build.hpp:168-272) -> dict of SoA arrays (parent, first_child, child_count,
    bmin, bmax, mean, scale, rot_wxyz, falloff, sh)."""
    cs = (or_camera * len(cams))(*[camera(c) for c in cams])
    out = C.c_void_p()
    _chk(lib().or_compact(oh.handle, cs, len(cams), float(tau_min), float(tau_max), C.byref(out)))
    try:
        n = int(lib().or_hierarchy_size(out))
        d = {"parent": np.empty(n, np.uint32), "first_child": np.empty(n, np.uint32),
             "child_count": np.empty(n, np.uint32), "bmin": np.empty((n, 3), np.float32),
             "bmax": np.empty((n, 3), np.float32), "mean": np.empty((n, 3), np.float32),
             "scale": np.empty((n, 3), np.float32), "rot_wxyz": np.empty((n, 4), np.float32),
             "falloff": np.empty(n, np.float32), "sh": np.empty((n, 48), np.float32)}
        lib().or_hierarchy_export(out, *[_p(d[k], C.c_uint32 if d[k].dtype == np.uint32 else C.c_float)
                                         for k in ("parent", "first_child", "child_count", "bmin", "bmax", "mean",
                                                   "scale", "rot_wxyz", "falloff", "sh")])
    finally:
        lib().or_hierarchy_free(out)
    return d


def render_backward(frame: OracleFrame, splats, cam, loss_grad, depth_grad=None, exposure=None) -> dict:
    """render_backward<float> (render.hpp:427-702) over `frame` (render_forward with keep_ctx)."""
    s, keep = _splats(splats)
    n = len(keep)
    lg = np.ascontiguousarray(loss_grad, np.float32)
    dg = None if depth_grad is None else np.ascontiguousarray(depth_grad, np.float32)
    ex = None if exposure is None else np.ascontiguousarray(exposure, np.float32).reshape(12)
    out = {"mean": np.zeros((n, 3), np.float32), "scale": np.zeros((n, 3), np.float32),
           "rotation": np.zeros((n, 4), np.float32), "falloff": np.zeros(n, np.float32),
           "parent_falloff": np.zeros(n, np.float32), "t": np.zeros(n, np.float32),
           "sh": np.zeros((n, 48), np.float32), "mean2d": np.zeros((n, 2), np.float32),
           "exposure": np.zeros((3, 4), np.float32)}
    _chk(lib().or_render_backward(frame.h, C.byref(s), n, C.byref(camera(cam)), _p(ex, C.c_float), _p(lg, C.c_float),
                                  _p(dg, C.c_float), *[_p(out[k], C.c_float) for k in
                                                       ("mean", "scale", "rotation", "falloff", "parent_falloff", "t",
                                                        "sh", "mean2d", "exposure")]))
    return out


def export_hierarchy(handle) -> dict:
    """An oracle Hierarchy handle -> SoA numpy arrays (or_hierarchy_export)."""
    n = int(lib().or_hierarchy_size(handle))
    d = dict(parent=np.empty(n, np.uint32), first_child=np.empty(n, np.uint32), child_count=np.empty(n, np.uint32),
             bmin=np.empty((n, 3), np.float32), bmax=np.empty((n, 3), np.float32), mean=np.empty((n, 3), np.float32),
             scale=np.empty((n, 3), np.float32), rot_wxyz=np.empty((n, 4), np.float32),
             falloff=np.empty(n, np.float32), sh=np.empty((n, 48), np.float32))
    lib().or_hierarchy_export(handle, *[_p(d[k], C.c_uint32) for k in ("parent", "first_child", "child_count")],
                              *[_p(d[k], C.c_float) for k in ("bmin", "bmax", "mean", "scale", "rot_wxyz",
                                                               "falloff", "sh")])
    return d


def photometric_loss(pred, target, want_grad=True):
    """photometric_loss (image.hpp:193-206) on (3, H, W) float32 images -> (loss, grad or None)."""
    p = np.ascontiguousarray(pred, np.float32)
    t = np.ascontiguousarray(target, np.float32)
    g = np.empty_like(p) if want_grad else None
    loss = float(lib().or_photometric_loss(_p(p, C.c_float), _p(t, C.c_float), p.shape[2], p.shape[1],
                                           _p(g, C.c_float)))
    return loss, g


def refine_hierarchy(oh: OracleHierarchy, cams, images, cfg: dict, exposures=None):
    """refine_hierarchy (refine.hpp:253-402) -> (refined SoA dict, per-step losses, max_screen_grad)."""
    nv = len(cams)
    cv = (or_camera * nv)(*[camera(c) for c in cams])
    imgs = [np.ascontiguousarray(im, np.float32) for im in images]
    ptrs = (f32p * nv)(*[_p(im, C.c_float) for im in imgs])
    ex = None if exposures is None else np.ascontiguousarray(exposures, np.float32).reshape(nv, 12)
    c = or_refine_config()
    for k in ("tau_min", "tau_max", "lr_mean", "lr_scale", "lr_rotation", "lr_falloff", "lr_sh"):
        setattr(c, k, float(cfg[k]))
    c.steps, c.rng_seed = int(cfg["steps"]), int(cfg.get("rng_seed", 0))
    loss = np.empty(max(1, c.steps), np.float64)
    mg = np.empty(oh.n, np.float32)
    out = _vp()
    _chk(lib().or_refine_hierarchy(oh.handle, cv, nv, ptrs, _p(ex, C.c_float), C.byref(c), C.byref(out),
                                   _p(loss, C.c_double), _p(mg, C.c_float)))
    try:
        d = export_hierarchy(out)
    finally:
        lib().or_hierarchy_free(out)
    return d, loss[:c.steps], mg
