"""Seeded fixtures mirroring /root/reference/proj/tests/support/fixtures.hpp
(random_gaussian :35-45, random_quat :28-33, look_at_camera :102-121) and the
scene/camera generators of tests/test_lod.cpp:35-51 and tests/test_render.cpp:44-67."""
import math

import numpy as np

import paper_2406_12080_b200 as hs


class Rng:
    def __init__(self, seed):
        self.g = np.random.default_rng(seed)

    def uniform(self, lo, hi, size=None):
        v = self.g.uniform(lo, hi, size)
        return np.float32(v) if size is None else v.astype(np.float32)

    def randint(self, n):
        return int(self.g.integers(0, n))

    def quat(self, n):
        q = self.g.normal(size=(n, 4)).astype(np.float32)
        q /= np.linalg.norm(q, axis=1, keepdims=True).astype(np.float32)
        return q.astype(np.float32)


def random_gaussians(rng, n, spread=2.0, smin=0.3, smax=1.5, fmin=0.1, fmax=1.0):
    """fixtures::random_gaussian x n -> (mean, scale, rot_wxyz, falloff, sh)."""
    mean = rng.uniform(-spread, spread, (n, 3))
    scale = rng.uniform(smin, smax, (n, 3))
    rot = rng.quat(n)
    fall = rng.uniform(fmin, fmax, n)
    sh = rng.uniform(-0.5, 0.5, (n, 48))
    return mean, scale, rot, fall, sh


def random_hierarchy(rng, n, spread=5.0):
    """test_lod.cpp:35-41."""
    return hs.build_bvh(*random_gaussians(rng, n, spread, 0.05, 0.5, 0.2, 1.0))


def random_camera(rng, scene_spread):
    """test_lod.cpp:43-51."""
    r = float(rng.uniform(0.5 * scene_spread, 6.0 * scene_spread))
    az = float(rng.uniform(0.0, 6.2831853))
    el = float(rng.uniform(-1.2, 1.2))
    pos = [r * math.cos(el) * math.cos(az), r * math.sin(el), r * math.cos(el) * math.sin(az)]
    target = rng.uniform(-0.3 * scene_spread, 0.3 * scene_spread, 3)
    w = 64 << rng.randint(4)
    h = 64 << rng.randint(4)
    return hs.look_at_camera(pos, target, w, h, float(rng.uniform(100.0, 600.0)))


def random_scene(rng, n, with_transitions):
    """test_render.cpp:44-56."""
    mean, scale, rot, fall, sh = random_gaussians(rng, n, 2.0, 0.05, 0.6)
    sp = hs.RenderSplats.plain(mean, scale, rot, sh, fall)
    if with_transitions:
        for i in range(n):
            if rng.randint(3) == 0:
                sp.t[i] = rng.uniform(0.05, 0.95)
                sp.parent_falloff[i] = rng.uniform(0.1, 1.0)
                sp.siblings[i] = 2 + rng.randint(3)
    return sp


def random_scene_camera(rng):
    """test_render.cpp:58-67 (odd sizes exercise partial tiles)."""
    az = float(rng.uniform(0.0, 6.2831853))
    el = float(rng.uniform(-0.9, 0.9))
    r = float(rng.uniform(6.0, 14.0))
    pos = [r * math.cos(el) * math.cos(az), r * math.sin(el), r * math.cos(el) * math.sin(az)]
    w = 48 + 16 * rng.randint(4)
    h = 40 + 8 * rng.randint(5)
    return hs.look_at_camera(pos, rng.uniform(-0.5, 0.5, 3), w, h, float(rng.uniform(40.0, 120.0)))


def axis_camera(w, h, focal):
    """test_render.cpp:19-21."""
    return hs.look_at_camera([0, 0, 0], [0, 0, 1], w, h, focal)


def gray_splat(mean, sigma, falloff):
    """test_render.cpp:36-42: flat 0.5 gray (SH all zero)."""
    return hs.RenderSplats.plain(np.asarray(mean, np.float32).reshape(1, 3), np.full((1, 3), sigma, np.float32),
                                 np.array([[1, 0, 0, 0]], np.float32), np.zeros((1, 48), np.float32),
                                 np.array([falloff], np.float32))


def concat(splats):
    fields = ["mean", "scale", "rot_wxyz", "sh", "falloff", "parent_falloff", "t", "siblings"]
    return hs.RenderSplats(*[np.concatenate([getattr(s, f) for s in splats]) for f in fields])


def descend(h, cam, tau, granularity):
    """Recursive-descent cut oracle (test_lod.cpp:18-26)."""
    out = []
    stack = [0]
    while stack:
        i = stack.pop()
        if granularity(h.bmin[i], h.bmax[i], cam) <= tau or h.child_count[i] == 0:
            out.append(i)
            continue
        fc, cc = int(h.first_child[i]), int(h.child_count[i])
        stack.extend(range(fc + cc - 1, fc - 1, -1))
    return sorted(out)
