"""B200-native hot path of arXiv 2406.12080 (hierarchical 3D Gaussians).

Host-side mirror of the reference library's public API for this path
(``hsplat`` namespace, /root/reference/proj/include/hsplat), backed by the C ABI
in include/hsplat_b200.h (libhsplat_b200.so, CUDA sm_100a):

==========================  ===============================================
reference (C++)             here
==========================  ===============================================
Hierarchy / read_hierarchy  Hierarchy, read_hierarchy, write_hierarchy
                            (model.hpp:93-139, io.hpp:342-408)
select_cut                  select_cut            (lod.hpp:52-92)
cut_render_splats           cut_render_splats     (lod.hpp:148-153)
render_forward              render_forward        (render.hpp:244-354)
render_hierarchy            render_hierarchy      (render.hpp:706-720)
bench_path                  bench_path            (bench.hpp:55-103)
read_cameras / camera path  read_cameras, read_camera_path (io.hpp:410-511)
psnr                        psnr                  (image.hpp:111-122)
hsplat::Error / Errc        Error / Errc          (errors.hpp)
==========================  ===============================================

Every compute call runs on the GPU through the C ABI; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

__all__ = [
    "Errc", "Error", "CameraModel", "Hierarchy", "CutEntries", "RenderSplats", "RenderOutput", "StageTimes",
    "FrameStats", "BenchReport", "Renderer", "DeviceHierarchy", "look_at_camera", "synth_city", "read_hierarchy",
    "write_hierarchy", "validate_hierarchy", "build_bvh", "read_cameras", "write_cameras", "read_camera_path",
    "write_camera_path", "select_cut", "cut_render_splats", "render_forward", "render_hierarchy", "bench_path",
    "psnr", "default_renderer", "NO_NODE",
]

NO_NODE = 0xFFFFFFFF
K_TILE = 16


class Errc(enum.IntEnum):
    """hsplat::Errc (errors.hpp:11-25); C-ABI status = value + 1."""
    AllZeroWeights = 0
    DegenerateCovariance = 1
    NotSPD = 2
    MissingForwardState = 3
    NoInteriorNodes = 4
    DegenerateSpread = 5
    MalformedHeader = 6
    TruncatedRecord = 7
    UnsupportedShDegree = 8
    EmptyScene = 9
    DimensionMismatch = 10
    InvalidArgument = 11
    IoFailure = 12


class Error(RuntimeError):
    """hsplat::Error: carries an Errc (or a device status); message prefixed with its name."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.code = Errc(status - 1) if 1 <= status <= 13 else None


def _check(status: int, ctx=None, what: str = ""):
    if status == 0:
        return
    if ctx is not None:
        msg = N.lib().hs_last_error(ctx).decode()
    else:
        msg = f"{N.lib().hs_status_name(status).decode()}: {what}"
    raise Error(status, msg)


# ----------------------------------------------------------------------------- camera
@dataclass
class CameraModel:
    """CameraModel (model.hpp:64-82): pinhole, world_to_camera [R|t] (3x4, float32)."""
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    world_to_camera: np.ndarray

    def to_c(self) -> N.hs_camera:
        c = N.hs_camera()
        c.width, c.height = int(self.width), int(self.height)
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        w = np.ascontiguousarray(self.world_to_camera, dtype=np.float32).reshape(12)
        for i in range(12):
            c.w2c[i] = float(w[i])
        return c

    def position(self) -> np.ndarray:
        r = self.world_to_camera[:, :3].astype(np.float32)
        t = self.world_to_camera[:, 3].astype(np.float32)
        return (-r.T) @ t


def _normalized(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.float32)
    n = np.float32(math.sqrt(float(np.dot(v, v))))
    return (v / n).astype(np.float32) if n > 0 else v


def look_at_camera(pos, target, width: int, height: int, focal: float, up=(0.0, 1.0, 0.0)) -> CameraModel:
    """fixtures::look_at_camera (tests/support/fixtures.hpp:102-121): +z forward, +x right."""
    pos = np.asarray(pos, dtype=np.float32)
    target = np.asarray(target, dtype=np.float32)
    up = np.asarray(up, dtype=np.float32)
    zc = _normalized(target - pos)
    xc = np.cross(up, zc).astype(np.float32)
    if float(np.linalg.norm(xc)) < 1e-5:
        xc = np.array([1.0, 0.0, 0.0], dtype=np.float32)
    xc = _normalized(xc)
    yc = np.cross(zc, xc).astype(np.float32)
    w2c = np.zeros((3, 4), dtype=np.float32)
    w2c[0, :3], w2c[1, :3], w2c[2, :3] = xc, yc, zc
    w2c[:, 3] = -(w2c[:, :3] @ pos)
    return CameraModel(width, height, focal, focal, width * 0.5, height * 0.5, w2c)


# ----------------------------------------------------------------------------- hierarchy
@dataclass
class Hierarchy:
    """Hierarchy (model.hpp:93-115) as host structure-of-arrays; root 0, children contiguous."""
    parent: np.ndarray       # u32 [N]
    first_child: np.ndarray  # u32 [N]
    child_count: np.ndarray  # u32 [N]
    bmin: np.ndarray         # f32 [N,3]
    bmax: np.ndarray         # f32 [N,3]
    mean: np.ndarray         # f32 [N,3]
    scale: np.ndarray        # f32 [N,3]
    rot_wxyz: np.ndarray     # f32 [N,4]
    falloff: np.ndarray      # f32 [N]
    sh: np.ndarray           # f32 [N,48]
    sh_degree: int = 3

    @property
    def n(self) -> int:
        return int(self.parent.shape[0])

    def leaf_count(self) -> int:
        return int(np.count_nonzero(self.child_count == 0))

    @staticmethod
    def empty(n: int) -> "Hierarchy":
        return Hierarchy(np.zeros(n, np.uint32), np.zeros(n, np.uint32), np.zeros(n, np.uint32),
                         np.zeros((n, 3), np.float32), np.zeros((n, 3), np.float32), np.zeros((n, 3), np.float32),
                         np.zeros((n, 3), np.float32), np.zeros((n, 4), np.float32), np.zeros(n, np.float32),
                         np.zeros((n, 48), np.float32))

    def contiguous(self) -> "Hierarchy":
        def c(a, dt):
            return np.ascontiguousarray(a, dtype=dt)
        return Hierarchy(c(self.parent, np.uint32), c(self.first_child, np.uint32), c(self.child_count, np.uint32),
                         c(self.bmin, np.float32), c(self.bmax, np.float32), c(self.mean, np.float32),
                         c(self.scale, np.float32), c(self.rot_wxyz, np.float32), c(self.falloff, np.float32),
                         c(self.sh, np.float32), self.sh_degree)

    def soa(self) -> N.hs_node_soa:
        s = N.hs_node_soa()
        s.parent, s.first_child, s.child_count = (N.ptr(self.parent, C.c_uint32), N.ptr(self.first_child, C.c_uint32),
                                                  N.ptr(self.child_count, C.c_uint32))
        s.bmin, s.bmax = N.ptr(self.bmin, C.c_float), N.ptr(self.bmax, C.c_float)
        s.mean, s.scale = N.ptr(self.mean, C.c_float), N.ptr(self.scale, C.c_float)
        s.rot_wxyz, s.falloff, s.sh = (N.ptr(self.rot_wxyz, C.c_float), N.ptr(self.falloff, C.c_float),
                                       N.ptr(self.sh, C.c_float))
        return s


def synth_city(leaves: int, seed: int = 1, threads: int = 0) -> Hierarchy:
    """Deterministic synthetic city hierarchy in build_bvh layout (csrc/synth.cpp)."""
    n = int(N.lib().hs_synth_node_count(leaves))
    h = Hierarchy.empty(n)
    _check(N.lib().hs_synth_city(leaves, seed, threads, C.byref(h.soa())), what="hs_synth_city")
    return h


def synth_city_chunk(leaves: int, seed: int, cx: float, cz: float, threads: int = 0) -> Hierarchy:
    """One chunk of a multi-chunk scene: synth_city statistics centred at (cx, 0, cz)."""
    n = int(N.lib().hs_synth_node_count(leaves))
    h = Hierarchy.empty(n)
    _check(N.lib().hs_synth_city_chunk(leaves, seed, float(cx), float(cz), threads, C.byref(h.soa())),
           what="hs_synth_city_chunk")
    return h


def synth_skybox(count: int, scene_diameter: float, seed: int = 0, centroid=(0.0, 0.0, 0.0),
                 threads: int = 0) -> Hierarchy:
    """make_skybox (scene.hpp:111-137) + build_bvh: mid-gray shell 5 diameters out."""
    n = int(N.lib().hs_synth_node_count(count))
    h = Hierarchy.empty(n)
    c = (C.c_float * 3)(*[float(v) for v in centroid])
    _check(N.lib().hs_synth_skybox(count, float(scene_diameter), seed, c, threads, C.byref(h.soa())),
           what="hs_synth_skybox")
    return h


def build_bvh(mean, scale, rot_wxyz, falloff, sh, threads: int = 0) -> Hierarchy:
    """build_bvh (build.hpp:73-149): median-split BVH + moment-matched interior nodes."""
    n = len(falloff)
    if n == 0:
        raise Error(int(Errc.EmptyScene) + 1, "EmptyScene: build_bvh needs at least one gaussian")
    a = [np.ascontiguousarray(x, np.float32).reshape(n, -1) for x in (mean, scale, rot_wxyz, falloff, sh)]
    h = Hierarchy.empty(2 * n - 1 if n else 0)
    st = N.lib().hs_build_bvh(*[N.ptr(x, C.c_float) for x in a], n, threads, C.byref(h.soa()))
    if st:
        name = N.lib().hs_status_name(st).decode()
        raise Error(st, f"{name}: build_bvh needs at least one gaussian with falloff in (0, 1] and scale > 0")
    return h


def scene_side(leaves: int) -> float:
    return float(N.lib().hs_synth_scene_side(leaves))


def validate_hierarchy(h: Hierarchy) -> None:
    """validate_hierarchy (model.hpp:118-139); raises Error(InvalidArgument)."""
    h = h.contiguous()
    buf = C.create_string_buffer(256)
    st = N.lib().hs_validate_hierarchy(C.byref(h.soa()), h.n, buf, 256)
    if st:
        raise Error(st, f"InvalidArgument: {buf.value.decode()}")


def read_hierarchy(path: str) -> Hierarchy:
    """read_hierarchy (io.hpp:375-408): .h3dg reader + validation."""
    n = C.c_uint64()
    deg = C.c_uint32()
    _check(N.lib().hs_h3dg_read_header(path.encode(), C.byref(n), C.byref(deg)), what=f"cannot read {path}")
    h = Hierarchy.empty(n.value)
    h.sh_degree = deg.value
    _check(N.lib().hs_h3dg_read(path.encode(), C.byref(h.soa()), n.value), what=f"cannot read {path}")
    validate_hierarchy(h)
    return h


def write_hierarchy(path: str, h: Hierarchy) -> None:
    """write_hierarchy (io.hpp:350-373)."""
    h = h.contiguous()
    _check(N.lib().hs_h3dg_write(path.encode(), C.byref(h.soa()), h.n, h.sh_degree), what=f"cannot write {path}")


# ----------------------------------------------------------------------------- camera text IO
def _cam_line(c: CameraModel, prec: int) -> str:
    vals = [c.width, c.height, c.fx, c.fy, c.cx, c.cy] + [float(v) for v in np.asarray(c.world_to_camera).reshape(12)]
    return " ".join(str(v) if isinstance(v, int) else f"{float(v):.{prec}g}" for v in vals)


def _data_lines(path: str):
    with open(path, "r") as f:
        for line in f.read().split("\n"):
            line = line.rstrip("\r")
            s = line.lstrip(" \t")
            if not s or s[0] == "#":
                continue
            yield line


def _parse_camera(tokens, line) -> CameraModel:
    if len(tokens) != 18:
        raise Error(int(Errc.MalformedHeader) + 1, f"MalformedHeader: expected 18 numbers per camera: {line}")
    try:
        w, h = int(tokens[0]), int(tokens[1])
        v = [np.float32(t) for t in tokens[2:]]
    except ValueError:
        raise Error(int(Errc.MalformedHeader) + 1, f"MalformedHeader: expected 18 numbers per camera: {line}")
    cam = CameraModel(w, h, v[0], v[1], v[2], v[3], np.array(v[4:], dtype=np.float32).reshape(3, 4))
    _validate_camera(cam)
    return cam


def _validate_camera(c: CameraModel) -> None:
    """validate_camera (model.hpp:84-91)."""
    def bad(msg):
        raise Error(int(Errc.InvalidArgument) + 1, f"InvalidArgument: {msg}")
    if not (c.width > 0 and c.height > 0):
        bad("camera resolution must be positive")
    if not (c.fx > 0 and c.fy > 0):
        bad("camera focal must be positive")
    w = np.asarray(c.world_to_camera, dtype=np.float32)
    if not np.all(np.isfinite(w)):
        bad("camera pose must be finite")
    r = w[:, :3]
    if not (np.linalg.norm(r @ r.T - np.eye(3, dtype=np.float32)) < 1e-3):
        bad("world_to_camera rotation block must be orthonormal")


def read_cameras(path: str) -> list[CameraModel]:
    """read_cameras (io.hpp:473-480)."""
    return [_parse_camera(line.split(), line) for line in _data_lines(path)]


def write_cameras(path: str, cams) -> None:
    with open(path, "w") as f:
        f.write("# width height fx fy cx cy  world-to-camera 3x4 row-major\n")
        for c in cams:
            f.write(_cam_line(c, 9) + "\n")


def read_camera_path(path: str) -> tuple[list[float], list[CameraModel]]:
    """read_camera_path (io.hpp:498-511): strictly increasing timestamps."""
    ts, cams = [], []
    for line in _data_lines(path):
        tok = line.split()
        try:
            t = float(tok[0])
        except (ValueError, IndexError):
            raise Error(int(Errc.MalformedHeader) + 1, f"MalformedHeader: expected a leading timestamp: {line}")
        cams.append(_parse_camera(tok[1:], line))
        if ts and not t > ts[-1]:
            raise Error(int(Errc.InvalidArgument) + 1, "InvalidArgument: timestamps must be strictly increasing")
        ts.append(t)
    return ts, cams


def write_camera_path(path: str, timestamps, cams) -> None:
    if len(timestamps) != len(cams):
        raise Error(int(Errc.DimensionMismatch) + 1, "DimensionMismatch: one timestamp per camera")
    for a, b in zip(timestamps, timestamps[1:]):
        if not b > a:
            raise Error(int(Errc.InvalidArgument) + 1, "InvalidArgument: timestamps must be strictly increasing")
    with open(path, "w") as f:
        f.write("# timestamp  width height fx fy cx cy  world-to-camera 3x4 row-major\n")
        for t, c in zip(timestamps, cams):
            f.write(f"{t:.17g} " + _cam_line(c, 9) + "\n")


# ----------------------------------------------------------------------------- results
@dataclass
class CutEntries:
    """std::vector<CutEntry> (model.hpp:144-148) as arrays, ascending node order."""
    node: np.ndarray
    t: np.ndarray
    alpha_prime: np.ndarray

    def __len__(self):
        return int(self.node.shape[0])


@dataclass
class RenderSplats:
    """std::vector<RenderSplat> (model.hpp:157-177) as arrays."""
    mean: np.ndarray
    scale: np.ndarray
    rot_wxyz: np.ndarray
    sh: np.ndarray
    falloff: np.ndarray
    parent_falloff: np.ndarray
    t: np.ndarray
    siblings: np.ndarray

    def __len__(self):
        return int(self.mean.shape[0])

    @staticmethod
    def empty(n: int) -> "RenderSplats":
        return RenderSplats(np.zeros((n, 3), np.float32), np.ones((n, 3), np.float32),
                            np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1)), np.zeros((n, 48), np.float32),
                            np.ones(n, np.float32), np.zeros(n, np.float32), np.ones(n, np.float32),
                            np.ones(n, np.int32))

    def contiguous(self) -> "RenderSplats":
        def c(a, dt):
            return np.ascontiguousarray(a, dtype=dt)
        return RenderSplats(c(self.mean, np.float32), c(self.scale, np.float32), c(self.rot_wxyz, np.float32),
                            c(self.sh, np.float32), c(self.falloff, np.float32), c(self.parent_falloff, np.float32),
                            c(self.t, np.float32), c(self.siblings, np.int32))

    def soa(self) -> N.hs_splat_soa:
        s = N.hs_splat_soa()
        s.mean, s.scale, s.rot_wxyz, s.sh = (N.ptr(self.mean, C.c_float), N.ptr(self.scale, C.c_float),
                                             N.ptr(self.rot_wxyz, C.c_float), N.ptr(self.sh, C.c_float))
        s.falloff, s.parent_falloff, s.t = (N.ptr(self.falloff, C.c_float), N.ptr(self.parent_falloff, C.c_float),
                                            N.ptr(self.t, C.c_float))
        s.siblings = N.ptr(self.siblings, C.c_int32)
        return s

    @staticmethod
    def plain(mean, scale, rot_wxyz, sh, falloff) -> "RenderSplats":
        """RenderSplat::plain (model.hpp:164-172) for arrays of Gaussians."""
        n = len(falloff)
        return RenderSplats(np.asarray(mean, np.float32).reshape(n, 3), np.asarray(scale, np.float32).reshape(n, 3),
                            np.asarray(rot_wxyz, np.float32).reshape(n, 4), np.asarray(sh, np.float32).reshape(n, 48),
                            np.asarray(falloff, np.float32), np.zeros(n, np.float32), np.ones(n, np.float32),
                            np.ones(n, np.int32))


@dataclass
class StageTimes:
    """StageTimes (render.hpp:24-31), seconds; `weights` is fused into preprocess on the GPU."""
    cut_expand: float = 0.0
    weights: float = 0.0
    preprocess: float = 0.0
    duplicate: float = 0.0
    tile_ranges: float = 0.0
    alpha_blend: float = 0.0

    def add(self, c: N.hs_stage_times):
        self.cut_expand += c.cut_expand
        self.weights += c.weights
        self.preprocess += c.preprocess
        self.duplicate += c.duplicate
        self.tile_ranges += c.tile_ranges
        self.alpha_blend += c.alpha_blend

    def total(self) -> float:
        return self.cut_expand + self.weights + self.preprocess + self.duplicate + self.tile_ranges + self.alpha_blend


@dataclass
class RenderOutput:
    """RenderOutput (render.hpp:77-83): planar images + rendered_count; `context` holds the
    ForwardContext parity view (tile_start, sorted keys/ids) when requested."""
    color: np.ndarray          # (3, H, W)
    depth: np.ndarray          # (H, W) blended inverse depth
    transmittance: np.ndarray  # (H, W)
    rendered_count: int
    info: dict = field(default_factory=dict)
    context: dict | None = None


# ----------------------------------------------------------------------------- device objects
class DeviceHierarchy:
    """Device-resident hierarchy (hs_hierarchy)."""

    def __init__(self, renderer: "Renderer", handle, n: int, leaves: int):
        self._r = renderer
        self.handle = handle
        self.n = n
        self.leaves = leaves

    def leaf_count(self) -> int:
        return self.leaves

    def __del__(self):
        try:
            if getattr(self, "handle", None) and N._lib is not None and self._r.ctx is not None:
                N.lib().hs_hierarchy_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class TransferTracker:
    """bench_path's cut-churn count (bench.hpp:79-82) on the device: count(cut)
    returns how many nodes of the renderer's current cut were absent from the
    cut passed to the previous count() call (all of them the first time)."""

    def __init__(self, renderer: "Renderer", dh: DeviceHierarchy):
        self.r = renderer
        self.dh = dh
        h = C.c_void_p()
        _check(N.lib().hs_transfer_tracker_create(renderer.ctx, dh.handle, C.byref(h)), renderer.ctx)
        self.handle = h

    def count(self, cut_handle=None) -> int:
        n = C.c_uint64()
        _check(N.lib().hs_transfer_count(self.r.ctx, self.handle, cut_handle or self.r._cut, C.byref(n)), self.r.ctx)
        return int(n.value)

    def close(self):
        if getattr(self, "handle", None) and getattr(self.r, "ctx", None):
            N.lib().hs_transfer_tracker_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class RefineConfig:
    """RefineConfig (refine.hpp:21-34)."""
    tau_min: float = 3.0
    tau_max: float = 48.0
    steps: int = 200
    lr_mean: float = 1.6e-5
    lr_scale: float = 5e-4
    lr_rotation: float = 1e-4
    lr_falloff: float = 5e-3
    lr_sh: float = 2.5e-4
    rng_seed: int = 0


@dataclass
class RefineStats:
    """RefineStats (refine.hpp:207-210): loss per step, per-node running max |d loss / d mean2d|."""
    loss: list
    max_screen_grad: np.ndarray


class Renderer:
    """One CUDA context (device, stream) running the hot path.  Mirrors the
    reference's free functions as methods; module-level wrappers use
    default_renderer()."""

    def __init__(self, device: int = 0, *, exact: bool = True, debug: bool = False, stats: bool = False):
        L = N.lib()
        h = C.c_void_p()
        _check(L.hs_context_create(device, C.byref(h)), what="hs_context_create (is a CUDA device visible?)")
        self.ctx = h
        self.device = device
        self.set_exact(exact)
        self.set_debug(debug)
        self.set_stats(stats)
        f = C.c_void_p()
        _check(L.hs_frame_create(self.ctx, C.byref(f)), self.ctx)
        self._frame = f
        c = C.c_void_p()
        _check(L.hs_cut_create(self.ctx, C.byref(c)), self.ctx)
        self._cut = c
        self._cache: dict = {}

    def close(self):
        L = N.lib()
        if getattr(self, "ctx", None):
            L.hs_frame_destroy(self._frame)
            L.hs_cut_destroy(self._cut)
            self._cache.clear()
            L.hs_context_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # options
    def set_exact(self, exact: bool):
        _check(N.lib().hs_context_set_option(self.ctx, N.HS_OPT_BLEND_MODE, 0 if exact else 1), self.ctx)

    def set_debug(self, debug: bool):
        self.debug = bool(debug)
        _check(N.lib().hs_context_set_option(self.ctx, N.HS_OPT_DEBUG, 1 if debug else 0), self.ctx)

    def set_stats(self, on: bool):
        """HS_OPT_STATS: the blend counts its work (info n_eval, n_eval_t, n_contrib, n_exp, n_pow)."""
        _check(N.lib().hs_context_set_option(self.ctx, N.HS_OPT_STATS, 1 if on else 0), self.ctx)

    def set_async(self, on: bool):
        _check(N.lib().hs_context_set_option(self.ctx, N.HS_OPT_ASYNC, 1 if on else 0), self.ctx)

    def set_lanes(self, n: int):
        """Frame lanes (HS_OPT_LANES): frame objects bind round-robin to n streams at
        their first render, so frames rendered on different objects overlap."""
        _check(N.lib().hs_context_set_option(self.ctx, N.HS_OPT_LANES, int(n)), self.ctx)

    def join(self):
        """Order the context stream after the work enqueued on every lane."""
        _check(N.lib().hs_context_join(self.ctx), self.ctx)

    def stream_handle(self) -> int:
        return int(N.lib().hs_context_stream(self.ctx) or 0)

    def synchronize(self):
        _check(N.lib().hs_context_synchronize(self.ctx), self.ctx)

    # hierarchy
    def upload(self, h: Hierarchy, validate: bool = True) -> DeviceHierarchy:
        h = h.contiguous()
        out = C.c_void_p()
        _check(N.lib().hs_hierarchy_upload(self.ctx, C.byref(h.soa()), h.n, h.sh_degree, 1 if validate else 0,
                                           C.byref(out)), self.ctx)
        return DeviceHierarchy(self, out, h.n, int(N.lib().hs_hierarchy_leaf_count(out)))

    def load_h3dg(self, path: str) -> DeviceHierarchy:
        out = C.c_void_p()
        _check(N.lib().hs_hierarchy_load_h3dg(self.ctx, path.encode(), C.byref(out)), self.ctx)
        return DeviceHierarchy(self, out, int(N.lib().hs_hierarchy_node_count(out)),
                               int(N.lib().hs_hierarchy_leaf_count(out)))

    def assemble(self, parts) -> DeviceHierarchy:
        """consolidate's global assembly (scene.hpp:228-316) on the device: the parts
        (chunk trees, then the skybox) under one merged root, serialised breadth-first."""
        devs = [self._dev(p) for p in parts]
        arr = (C.c_void_p * max(1, len(devs)))(*[d.handle for d in devs])
        out = C.c_void_p()
        _check(N.lib().hs_hierarchy_assemble(self.ctx, arr, len(devs), C.byref(out)), self.ctx)
        return DeviceHierarchy(self, out, int(N.lib().hs_hierarchy_node_count(out)),
                               int(N.lib().hs_hierarchy_leaf_count(out)))

    def compact(self, h, cams, tau_min: float = 3.0, tau_max: float = 0.0) -> DeviceHierarchy:
        """compact (build.hpp:168-272) on the device: a new, breadth-first hierarchy without the
        interior nodes no probed cut of `cams` uses."""
        dh = self._dev(h)
        cc = (N.hs_camera * max(1, len(cams)))(*[c.to_c() for c in cams])
        out = C.c_void_p()
        _check(N.lib().hs_hierarchy_compact(self.ctx, dh.handle, cc, len(cams), float(tau_min), float(tau_max),
                                            C.byref(out)), self.ctx)
        return DeviceHierarchy(self, out, int(N.lib().hs_hierarchy_node_count(out)),
                               int(N.lib().hs_hierarchy_leaf_count(out)))

    def download(self, h) -> Hierarchy:
        """Device hierarchy -> host Hierarchy (reference node order)."""
        dh = self._dev(h)
        out = Hierarchy.empty(dh.n)
        _check(N.lib().hs_hierarchy_download(self.ctx, dh.handle, C.byref(out.soa())), self.ctx)
        return out

    def refine_hierarchy(self, h, cams, images, config: RefineConfig | None = None, exposures=None):
        """refine_hierarchy (refine.hpp:253-402) on the device: SGD over the interior nodes
        against the training views (images[v]: (3, H, W) of cams[v]).  Returns (refined
        DeviceHierarchy, RefineStats).  exposures: (n_views, 3, 4) or None (identity)."""
        cfg = config or RefineConfig()
        dh = self._dev(h)
        nv = len(cams)
        if nv != len(images):
            raise Error(int(Errc.DimensionMismatch) + 1, "DimensionMismatch: need one training image per camera")
        cc = (N.hs_camera * max(1, nv))(*[c.to_c() for c in cams])
        imgs = []
        for c, im in zip(cams, images):
            a = np.ascontiguousarray(im, np.float32)
            if a.shape != (3, c.height, c.width):
                raise Error(int(Errc.DimensionMismatch) + 1,
                            "DimensionMismatch: training image shape must match its camera")
            imgs.append(a)
        ptrs = (N.f32p * max(1, nv))(*[N.ptr(a, C.c_float) for a in imgs])
        ex = None if exposures is None else np.ascontiguousarray(exposures, np.float32).reshape(nv, 12)
        c = N.hs_refine_config(cfg.tau_min, cfg.tau_max, cfg.steps, cfg.lr_mean, cfg.lr_scale, cfg.lr_rotation,
                               cfg.lr_falloff, cfg.lr_sh, cfg.rng_seed)
        loss = np.zeros(max(1, cfg.steps), np.float64)
        mg = np.zeros(dh.n, np.float32)
        out = C.c_void_p()
        _check(N.lib().hs_refine_hierarchy(self.ctx, dh.handle, cc, ptrs, N.ptr(ex, C.c_float), nv, C.byref(c),
                                           C.byref(out), loss.ctypes.data_as(C.POINTER(C.c_double)),
                                           N.ptr(mg, C.c_float)), self.ctx)
        refined = DeviceHierarchy(self, out, dh.n, int(N.lib().hs_hierarchy_leaf_count(out)))
        return refined, RefineStats(list(loss[:cfg.steps]), mg)

    def photometric_loss(self, pred, target):
        """photometric_loss (image.hpp:193-206) on (3, H, W) images -> (loss, d loss / d pred)."""
        p = np.ascontiguousarray(pred, np.float32)
        t = np.ascontiguousarray(target, np.float32)
        g = np.empty_like(p)
        loss = C.c_float()
        _check(N.lib().hs_photometric_loss(self.ctx, N.ptr(p, C.c_float), N.ptr(t, C.c_float), p.shape[2],
                                           p.shape[1], C.byref(loss), N.ptr(g, C.c_float)), self.ctx)
        return float(loss.value), g

    def _dev(self, h) -> DeviceHierarchy:
        if isinstance(h, DeviceHierarchy):
            return h
        key = id(h)
        ent = self._cache.get(key)
        if ent is None or ent[0] is not h:
            self._cache[key] = (h, self.upload(h))
        return self._cache[key][1]

    # cut
    def _cut_arrays(self, cut_handle) -> CutEntries:
        n = C.c_uint64()
        _check(N.lib().hs_cut_size(self.ctx, cut_handle, C.byref(n)), self.ctx)
        node = np.empty(n.value, np.uint32)
        t = np.empty(n.value, np.float32)
        a = np.empty(n.value, np.float32)
        _check(N.lib().hs_cut_download(self.ctx, cut_handle, N.ptr(node, C.c_uint32), N.ptr(t, C.c_float),
                                       N.ptr(a, C.c_float)), self.ctx)
        return CutEntries(node, t, a)

    def select_cut(self, h, cam: CameraModel, tau: float) -> CutEntries:
        dh = self._dev(h)
        _check(N.lib().hs_select_cut(self.ctx, dh.handle, C.byref(cam.to_c()), float(tau), self._cut), self.ctx)
        return self._cut_arrays(self._cut)

    def select_cut_device(self, h, cam: CameraModel, tau: float) -> int:
        """select_cut keeping the entries on the device (the renderer's current cut); returns its size."""
        dh = self._dev(h)
        _check(N.lib().hs_select_cut(self.ctx, dh.handle, C.byref(cam.to_c()), float(tau), self._cut), self.ctx)
        n = C.c_uint64()
        _check(N.lib().hs_cut_size(self.ctx, self._cut, C.byref(n)), self.ctx)
        return int(n.value)

    def transfer_tracker(self, h) -> "TransferTracker":
        return TransferTracker(self, self._dev(h))

    def _install_cut(self, dh: DeviceHierarchy, cut: CutEntries):
        node = np.ascontiguousarray(cut.node, np.uint32)
        t = np.ascontiguousarray(cut.t, np.float32)
        a = np.ascontiguousarray(cut.alpha_prime, np.float32)
        _check(N.lib().hs_cut_upload(self.ctx, dh.handle, N.ptr(node, C.c_uint32), N.ptr(t, C.c_float),
                                     N.ptr(a, C.c_float), len(node), self._cut), self.ctx)

    def cut_render_splats(self, h, cut: CutEntries) -> RenderSplats:
        dh = self._dev(h)
        self._install_cut(dh, cut)
        out = RenderSplats.empty(len(cut))
        _check(N.lib().hs_cut_render_splats(self.ctx, dh.handle, self._cut, C.byref(out.soa())), self.ctx)
        return out

    # per-object API (lod.hpp:18-146, render.hpp:104-176): batch kernels on the device
    def granularity(self, bmin, bmax, cam: CameraModel) -> np.ndarray:
        """granularity (lod.hpp:18-26) of boxes bmin/bmax (n, 3)."""
        bmin = np.ascontiguousarray(bmin, np.float32).reshape(-1, 3)
        bmax = np.ascontiguousarray(bmax, np.float32).reshape(-1, 3)
        out = np.empty(len(bmin), np.float32)
        _check(N.lib().hs_granularity(self.ctx, N.ptr(bmin, C.c_float), N.ptr(bmax, C.c_float), len(bmin),
                                      C.byref(cam.to_c()), N.ptr(out, C.c_float)), self.ctx)
        return out

    def interp_weight(self, eps_node, eps_parent, tau: float) -> np.ndarray:
        """interp_weight (lod.hpp:34-37), element-wise."""
        en = np.ascontiguousarray(eps_node, np.float32).ravel()
        ep = np.ascontiguousarray(eps_parent, np.float32).ravel()
        out = np.empty(len(en), np.float32)
        _check(N.lib().hs_interp_weight(self.ctx, N.ptr(en, C.c_float), N.ptr(ep, C.c_float), len(en), float(tau),
                                        N.ptr(out, C.c_float)), self.ctx)
        return out

    def transition_alpha(self, parent_alpha, siblings) -> np.ndarray:
        """transition_alpha (lod.hpp:41-45), element-wise; InvalidArgument if any K < 1."""
        a = np.ascontiguousarray(parent_alpha, np.float32).ravel()
        k = np.ascontiguousarray(np.broadcast_to(siblings, a.shape), np.int32).ravel()
        out = np.empty(len(a), np.float32)
        _check(N.lib().hs_transition_alpha(self.ctx, N.ptr(a, C.c_float), N.ptr(k, C.c_int32), len(a),
                                           N.ptr(out, C.c_float)), self.ctx)
        return out

    @staticmethod
    def _gsoa(g: dict):
        arrs = {k: np.ascontiguousarray(g[k], np.float32) for k in ("mean", "scale", "rot_wxyz", "falloff", "sh")}
        s = N.hs_gaussian_soa(*[N.ptr(arrs[k], C.c_float) for k in ("mean", "scale", "rot_wxyz", "falloff", "sh")])
        return s, arrs

    def interpolated_gaussian(self, child: dict, parent: dict, t, siblings) -> dict:
        """interpolated_gaussian (lod.hpp:97-110) for arrays of Gaussians (dicts of mean (n,3),
        scale (n,3), rot_wxyz (n,4), falloff (n,), sh (n,48))."""
        sc, keep_c = self._gsoa(child)
        sp, keep_p = self._gsoa(parent)
        n = len(keep_c["falloff"])
        tt = np.ascontiguousarray(np.broadcast_to(t, (n,)), np.float32)
        k = np.ascontiguousarray(np.broadcast_to(siblings, (n,)), np.int32)
        out = {"mean": np.empty((n, 3), np.float32), "scale": np.empty((n, 3), np.float32),
               "rot_wxyz": np.empty((n, 4), np.float32), "falloff": np.empty(n, np.float32),
               "sh": np.empty((n, 48), np.float32)}
        so = N.hs_gaussian_soa(*[N.ptr(out[kk], C.c_float) for kk in ("mean", "scale", "rot_wxyz", "falloff", "sh")])
        _check(N.lib().hs_interpolated_gaussians(self.ctx, C.byref(sc), C.byref(sp), N.ptr(tt, C.c_float),
                                                 N.ptr(k, C.c_int32), n, C.byref(so)), self.ctx)
        return out

    def assemble_cut_splats(self, h, attrs: dict, cut: CutEntries) -> RenderSplats:
        """assemble_cut_splats (lod.hpp:116-146) over caller attribute arrays parallel to the nodes."""
        dh = self._dev(h)
        sa, keep = self._gsoa(attrs)
        node = np.ascontiguousarray(cut.node, np.uint32)
        t = np.ascontiguousarray(cut.t, np.float32)
        out = RenderSplats.empty(len(node))
        _check(N.lib().hs_assemble_cut_splats(self.ctx, dh.handle, C.byref(sa), len(keep["falloff"]),
                                              N.ptr(node, C.c_uint32), N.ptr(t, C.c_float), len(node),
                                              C.byref(out.soa())), self.ctx)
        return out

    def project(self, splats: RenderSplats, cam: CameraModel) -> np.ndarray:
        """project (render.hpp:104-176) of every splat: a structured array of ProjectedSplat fields."""
        sp = splats.contiguous()
        out = (N.hs_projected * max(1, len(sp)))()
        if len(sp):
            _check(N.lib().hs_project(self.ctx, C.byref(sp.soa()), len(sp), C.byref(cam.to_c()), out), self.ctx)
        return np.ctypeslib.as_array(out)[: len(sp)].copy()

    def render_reference(self, splats: RenderSplats, cam: CameraModel) -> RenderOutput:
        """render_reference (render.hpp:360-408): naive per-pixel walk over the whole depth order."""
        sp = splats.contiguous()
        _check(N.lib().hs_render_reference(self.ctx, C.byref(sp.soa()) if len(sp) else None, len(sp),
                                           C.byref(cam.to_c()), self._frame), self.ctx)
        return self._output(False)

    def frame_order(self) -> np.ndarray:
        """ForwardContext::order (render.hpp:93) of the last render: visible ids in depth order."""
        n = C.c_uint64()
        _check(N.lib().hs_frame_order(self.ctx, self._frame, None, C.byref(n)), self.ctx)
        o = np.empty(n.value, np.uint32)
        _check(N.lib().hs_frame_order(self.ctx, self._frame, N.ptr(o, C.c_uint32), C.byref(n)), self.ctx)
        return o

    # render
    def _output(self, want_context: bool) -> RenderOutput:
        L = N.lib()
        info = N.hs_frame_info()
        _check(L.hs_frame_get_info(self.ctx, self._frame, C.byref(info)), self.ctx)
        H, W = info.height, info.width
        color = np.empty((3, H, W), np.float32)
        depth = np.empty((H, W), np.float32)
        trans = np.empty((H, W), np.float32)
        rc = C.c_int32()
        _check(L.hs_frame_download(self.ctx, self._frame, N.ptr(color, C.c_float), N.ptr(depth, C.c_float),
                                   N.ptr(trans, C.c_float), C.byref(rc)), self.ctx)
        d = dict(width=W, height=H, tiles_x=info.tiles_x, tiles_y=info.tiles_y, n_splats=int(info.n_splats),
                 n_visible=int(info.n_visible), n_duplicates=int(info.n_duplicates), sort_passes=info.sort_passes,
                 n_eval=int(info.n_eval), n_contrib=int(info.n_contrib))
        out = RenderOutput(color, depth, trans, int(rc.value), d)
        if want_context:
            out.context = self.frame_debug(d)
        return out

    def frame_debug(self, info: dict | None = None) -> dict:
        """ForwardContext parity view: tile_start, sorted (key, id) list, and with debug on the
        pre-sort duplicated list and per-splat projection dumps."""
        L = N.lib()
        if info is None:
            fi = N.hs_frame_info()
            _check(L.hs_frame_get_info(self.ctx, self._frame, C.byref(fi)), self.ctx)
            info = dict(tiles_x=fi.tiles_x, tiles_y=fi.tiles_y, n_duplicates=int(fi.n_duplicates),
                        n_splats=int(fi.n_splats))
        tiles = info["tiles_x"] * info["tiles_y"]
        D = info["n_duplicates"]
        ts = np.empty(tiles + 1, np.uint64)
        keys = np.empty(D, np.uint64)
        vals = np.empty(D, np.uint32)
        dk = dv = pj = None
        if self.debug:
            dk = np.empty(D, np.uint64)
            dv = np.empty(D, np.uint32)
            pj = np.empty((info["n_splats"], 16), np.float32)
        _check(L.hs_frame_debug(self.ctx, self._frame, N.ptr(ts, C.c_uint64), N.ptr(keys, C.c_uint64),
                                N.ptr(vals, C.c_uint32), N.ptr(dk, C.c_uint64), N.ptr(dv, C.c_uint32),
                                N.ptr(pj, C.c_float)), self.ctx)
        return dict(tile_start=ts, sorted_keys=keys, sorted_vals=vals, dup_keys=dk, dup_vals=dv, proj16=pj,
                    order=self.frame_order())

    def render_forward(self, splats: RenderSplats, cam: CameraModel, *, want_context: bool = False,
                       stages: StageTimes | None = None) -> RenderOutput:
        sp = splats.contiguous()
        st = N.hs_stage_times()
        _check(N.lib().hs_render_splats(self.ctx, C.byref(sp.soa()) if len(sp) else None, len(sp),
                                        C.byref(cam.to_c()), self._frame, C.byref(st) if stages else None),
               self.ctx)
        if stages is not None:
            stages.add(st)
        return self._output(want_context)

    def render_backward(self, loss_grad, depth_grad=None, exposure=None) -> dict:
        """render_backward<float> (render.hpp:427-702) over the context of the last
        render_forward of this renderer: gradients w.r.t. every splat attribute and the
        exposure matrix (3x4), for loss_grad (3, H, W) w.r.t. the exposed colour."""
        fi = N.hs_frame_info()
        _check(N.lib().hs_frame_get_info(self.ctx, self._frame, C.byref(fi)), self.ctx)
        n, H, W = int(fi.n_splats), int(fi.height), int(fi.width)
        lg = np.ascontiguousarray(loss_grad, np.float32)
        if lg.shape != (3, H, W):
            raise Error(int(Errc.DimensionMismatch) + 1, "DimensionMismatch: loss gradient must be H x W x 3")
        dg = None
        if depth_grad is not None:
            dg = np.ascontiguousarray(depth_grad, np.float32)
            if dg.shape != (H, W):
                raise Error(int(Errc.DimensionMismatch) + 1, "DimensionMismatch: depth gradient must be H x W x 1")
        ex = None if exposure is None else np.ascontiguousarray(exposure, np.float32).reshape(12)
        out = {"mean": np.zeros((n, 3), np.float32), "scale": np.zeros((n, 3), np.float32),
               "rotation": np.zeros((n, 4), np.float32), "falloff": np.zeros(n, np.float32),
               "parent_falloff": np.zeros(n, np.float32), "t": np.zeros(n, np.float32),
               "sh": np.zeros((n, 48), np.float32), "mean2d": np.zeros((n, 2), np.float32),
               "exposure": np.zeros((3, 4), np.float32)}
        go = N.hs_grads_out(*[N.ptr(out[k], C.c_float) for k in ("mean", "scale", "rotation", "falloff",
                                                                  "parent_falloff", "t", "sh", "mean2d", "exposure")])
        _check(N.lib().hs_render_backward(self.ctx, self._frame, N.ptr(lg, C.c_float), N.ptr(dg, C.c_float),
                                          N.ptr(ex, C.c_float), C.byref(go)), self.ctx)
        return out

    def render_hierarchy(self, h, cam: CameraModel, tau: float, *, want_context: bool = False,
                         stages: StageTimes | None = None, return_cut: bool = False):
        dh = self._dev(h)
        st = N.hs_stage_times()
        _check(N.lib().hs_render_hierarchy(self.ctx, dh.handle, C.byref(cam.to_c()), float(tau), self._cut,
                                           self._frame, C.byref(st) if stages else None), self.ctx)
        if stages is not None:
            stages.add(st)
        out = self._output(want_context)
        if return_cut:
            return out, self._cut_arrays(self._cut)
        return out

    def render_cut(self, h, cam: CameraModel, *, stages: StageTimes | None = None) -> RenderOutput:
        """Render the cut selected by the last select_cut/render_hierarchy (bench.hpp:84 odd frames)."""
        dh = self._dev(h)
        st = N.hs_stage_times()
        _check(N.lib().hs_render_cut(self.ctx, dh.handle, self._cut, C.byref(cam.to_c()), self._frame,
                                     C.byref(st) if stages else None), self.ctx)
        if stages is not None:
            stages.add(st)
        return self._output(False)


_default: dict[int, Renderer] = {}


def default_renderer(device: int = 0) -> Renderer:
    r = _default.get(device)
    if r is None:
        r = _default[device] = Renderer(device)
    return r


# ----------------------------------------------------------------------------- free functions
def select_cut(h, cam: CameraModel, tau: float) -> CutEntries:
    """select_cut (lod.hpp:52-92)."""
    return default_renderer().select_cut(h, cam, tau)


def cut_render_splats(h, cut: CutEntries) -> RenderSplats:
    """cut_render_splats (lod.hpp:148-153)."""
    return default_renderer().cut_render_splats(h, cut)


def granularity(bmin, bmax, cam: CameraModel):
    """granularity (lod.hpp:18-26) of one box (bmin, bmax 3-vectors) or of arrays of boxes."""
    out = default_renderer().granularity(bmin, bmax, cam)
    return float(out[0]) if np.asarray(bmin).ndim == 1 else out


def interp_weight(eps_node, eps_parent, tau: float):
    """interp_weight (lod.hpp:34-37)."""
    out = default_renderer().interp_weight(eps_node, eps_parent, tau)
    return float(out[0]) if np.ndim(eps_node) == 0 else out


def transition_alpha(parent_alpha, siblings):
    """transition_alpha (lod.hpp:41-45)."""
    out = default_renderer().transition_alpha(parent_alpha, siblings)
    return float(out[0]) if np.ndim(parent_alpha) == 0 else out


def interpolated_gaussian(child: dict, parent: dict, t, siblings) -> dict:
    """interpolated_gaussian (lod.hpp:97-110)."""
    return default_renderer().interpolated_gaussian(child, parent, t, siblings)


def assemble_cut_splats(h, attrs: dict, cut: CutEntries) -> RenderSplats:
    """assemble_cut_splats<float> (lod.hpp:116-146)."""
    return default_renderer().assemble_cut_splats(h, attrs, cut)


def project(splats: RenderSplats, cam: CameraModel) -> np.ndarray:
    """project (render.hpp:104-176)."""
    return default_renderer().project(splats, cam)


def render_reference(splats: RenderSplats, cam: CameraModel) -> RenderOutput:
    """render_reference (render.hpp:360-408)."""
    return default_renderer().render_reference(splats, cam)


def set_thread_count(n: int) -> None:
    """set_thread_count (parallel.hpp:18): the CPU worker count of the reference; the GPU
    path has no host worker pool, so it changes nothing (results never depend on it)."""
    global _thread_count
    _thread_count = int(n)


_thread_count = 0


def render_forward(splats: RenderSplats, cam: CameraModel, ctx_out: dict | None = None,
                   stages: StageTimes | None = None) -> RenderOutput:
    """render_forward<float> (render.hpp:244-354); ctx_out receives the ForwardContext parity view."""
    out = default_renderer().render_forward(splats, cam, want_context=ctx_out is not None, stages=stages)
    if ctx_out is not None:
        ctx_out.update(out.context)
    return out


def render_backward(loss_grad, depth_grad=None, exposure=None) -> dict:
    """render_backward<float> (render.hpp:427-702) over the last render_forward of the default renderer."""
    return default_renderer().render_backward(loss_grad, depth_grad, exposure)


def render_hierarchy(h, cam: CameraModel, tau: float, ctx_out: dict | None = None,
                     stages: StageTimes | None = None) -> RenderOutput:
    """render_hierarchy (render.hpp:706-720)."""
    out = default_renderer().render_hierarchy(h, cam, tau, want_context=ctx_out is not None, stages=stages)
    if ctx_out is not None:
        ctx_out.update(out.context)
    return out


@dataclass
class FrameStats:
    """FrameStats (bench.hpp:17-22)."""
    rendered: int = 0
    rendered_pct: float = 0.0
    transferred: int = 0
    stages: StageTimes = field(default_factory=StageTimes)


@dataclass
class BenchReport:
    """BenchReport (bench.hpp:24-49)."""
    leaf_count: int = 0
    tau: float = 0.0
    frames: list = field(default_factory=list)
    mean_rendered: float = 0.0
    mean_rendered_pct: float = 0.0
    total_transferred: int = 0
    total_stages: StageTimes = field(default_factory=StageTimes)

    def csv(self) -> str:
        def row(label, rendered, pct, transferred, t):
            return (f"{label},{_fmt(rendered)},{_fmt(pct)},{transferred},{_fmt(t.cut_expand)},{_fmt(t.weights)},"
                    f"{_fmt(t.preprocess)},{_fmt(t.duplicate)},{_fmt(t.tile_ranges)},{_fmt(t.alpha_blend)}\n")
        s = ("frame,rendered,rendered_pct,transferred,cut_expand_s,weights_s,preprocess_s,duplicate_s,"
             "tile_ranges_s,alpha_blend_s\n")
        for i, f in enumerate(self.frames):
            s += row(str(i), f.rendered, f.rendered_pct, f.transferred, f.stages)
        s += row("total", self.mean_rendered, self.mean_rendered_pct, self.total_transferred, self.total_stages)
        return s


def _fmt(v) -> str:
    # std::ostream default formatting of a double (%g with 6 significant digits)
    return f"{float(v):g}"


def bench_path(h, cameras, tau: float, timestamps=None, renderer: Renderer | None = None) -> BenchReport:
    """bench_path (bench.hpp:55-103): cut refreshed on even frames and reused on odd
    ones; `transferred` counts cut nodes absent from the previous refresh."""
    r = renderer or default_renderer()
    if len(cameras) == 0:
        raise Error(int(Errc.InvalidArgument) + 1, "InvalidArgument: camera path is empty")
    if timestamps is not None and len(timestamps) not in (0, len(cameras)):
        raise Error(int(Errc.DimensionMismatch) + 1, "DimensionMismatch: one timestamp per camera")
    dh = r._dev(h)
    rep = BenchReport(leaf_count=dh.leaf_count(), tau=float(tau))
    tracker = r.transfer_tracker(dh)  # |cut \ previous cut| on the device
    cut_size = 0
    for i, cam in enumerate(cameras):
        fs = FrameStats()
        if i % 2 == 0:
            out = r.render_hierarchy(dh, cam, tau, stages=fs.stages)
            n = C.c_uint64()
            _check(N.lib().hs_cut_size(r.ctx, r._cut, C.byref(n)), r.ctx)
            cut_size = int(n.value)
            fs.transferred = tracker.count()
        else:
            out = r.render_cut(dh, cam, stages=fs.stages)
        del out
        fs.rendered = cut_size
        fs.rendered_pct = 100.0 * cut_size / rep.leaf_count
        rep.mean_rendered += fs.rendered
        rep.mean_rendered_pct += fs.rendered_pct
        rep.total_transferred += fs.transferred
        for k in ("cut_expand", "weights", "preprocess", "duplicate", "tile_ranges", "alpha_blend"):
            setattr(rep.total_stages, k, getattr(rep.total_stages, k) + getattr(fs.stages, k))
        rep.frames.append(fs)
    tracker.close()
    rep.mean_rendered /= len(rep.frames)
    rep.mean_rendered_pct /= len(rep.frames)
    return rep


def refine_hierarchy(h, cams, images, config: RefineConfig | None = None, exposures=None):
    """refine_hierarchy (refine.hpp:253-402) -> (refined Hierarchy, RefineStats)."""
    r = default_renderer()
    dh, stats = r.refine_hierarchy(h, cams, images, config, exposures)
    return r.download(dh), stats


def photometric_loss(pred, target):
    """photometric_loss (image.hpp:193-206) -> (loss, d loss / d pred)."""
    return default_renderer().photometric_loss(pred, target)


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    """psnr (image.hpp:111-122): all channels in double, mse <= 0 -> 99 dB, capped at 99."""
    if a.shape != b.shape:
        raise Error(int(Errc.DimensionMismatch) + 1, "DimensionMismatch: images must have identical shapes")
    d = a.astype(np.float64).ravel() - b.astype(np.float64).ravel()
    mse = float(np.dot(d, d)) / d.size
    if mse <= 0.0:
        return 99.0
    return float(np.float32(min(99.0, -10.0 * math.log10(mse))))
