"""Synthetic benchmark inputs: the BASELINE.json configurations.

Hierarchies come from csrc/synth.cpp (build_bvh layout).  Cameras fly a
closed loop around the outside of the city at a fixed altitude and stand-off
from its edge, always looking inward and down.  Keeping every camera outside
the scene with its view direction inside the inward cone guarantees that no
geometry lies near the camera's image plane: the reference renderer only culls
at z <= 0.01 (render.hpp:110) and has no frustum guard band, so a splat just in
front of the image plane projects to a screen-covering ellipse; a camera
inside the point cloud would render mostly those.  The near half of the city
is within the leaf-level LOD range, the far half is coarse, so the cut mixes
leaves, interior nodes and transitions as the paper's Table 5 paths do.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import CameraModel, look_at_camera, scene_side, synth_city, synth_city_chunk, synth_skybox


@dataclass(frozen=True)
class Config:
    name: str
    leaves: int
    width: int
    height: int
    focal: float
    tau: float
    altitude: float = 40.0
    standoff: float = 30.0
    lookahead: float = 150.0
    sky: int = 0  # multi-chunk scenes: make_skybox splats under the global root (0: none)


CONFIGS = {
    # BASELINE.json configs[0]: 100K leaves, single 640x480 view, tau = 3 px (CPU reference runs it)
    "c1": Config("c1_100k_640x480_tau3", 100_000, 640, 480, 300.0, 3.0, altitude=15.0, standoff=10.0,
                 lookahead=50.0),
    # configs[1]: 10M leaves, 1920x1080, tau = 3 px, 1 B200 (the headline metric)
    "c2": Config("c2_10m_1080p_tau3", 10_000_000, 1920, 1080, 1100.0, 3.0),
    # configs[4]: 100M leaves multi-chunk (4 x 4 chunks of 6.25M leaves, a km-scale city, under one
    # merged root, assembled breadth-first on the device: multichunk()), 3840x2160; ~58 GB resident
    "c5": Config("c5_100m_2160p_tau3", 100_000_000, 3840, 2160, 2200.0, 3.0, altitude=60.0, standoff=40.0,
                 lookahead=250.0),
    # C5 with the 100K-splat make_skybox shell (scene.hpp:111-137) under the global root.  The
    # reference projects shell splats lying just in front of the camera's image plane (at ~28 km
    # to the side) into screen-covering ellipses -- it culls only at z <= 0.01 (render.hpp:110)
    # and its EWA Jacobian has no field-of-view clamp -- and they sort first: every pixel
    # saturates on them and the city is hidden.  Rendered bit-exactly, reported separately.
    "c5sky": Config("c5sky_100m_2160p_tau3", 100_000_000, 3840, 2160, 2200.0, 3.0, altitude=60.0, standoff=40.0,
                    lookahead=250.0, sky=100_000),
}


def trajectory(cfg: Config, n_frames: int, first: int = 0) -> list[CameraModel]:
    """Frames [first, first + n_frames) of a closed loop of `1000` frames by default period."""
    side = scene_side(cfg.leaves)
    half = 0.5 * side + cfg.standoff
    period = 1000
    cams = []
    for i in range(first, first + n_frames):
        u = (i % period) / period * 4.0  # 4 edges, parameter along the square loop
        edge = int(u) % 4
        s = u - int(u)
        # square corners counter-clockwise starting at the south-west corner
        corners = [(-half, -half), (half, -half), (half, half), (-half, half)]
        x0, z0 = corners[edge]
        x1, z1 = corners[(edge + 1) % 4]
        px, pz = x0 + (x1 - x0) * s, z0 + (z1 - z0) * s
        # inward normals of the south, east, north, west edges; blend near corners
        normals = [(0.0, 1.0), (-1.0, 0.0), (0.0, -1.0), (1.0, 0.0)]
        n0 = np.array(normals[edge])
        w = 0.0
        if s > 0.9:
            w = (s - 0.9) / 0.2
            n1 = np.array(normals[(edge + 1) % 4])
        elif s < 0.1:
            w = (0.1 - s) / 0.2
            n1 = np.array(normals[(edge - 1) % 4])
        d = n0 if w == 0.0 else (1 - w) * n0 + w * n1
        d = d / np.linalg.norm(d)
        pos = np.array([px, cfg.altitude, pz], np.float32)
        target = np.array([px + d[0] * cfg.lookahead, 0.0, pz + d[1] * cfg.lookahead], np.float32)
        cams.append(look_at_camera(pos, target, cfg.width, cfg.height, cfg.focal))
    return cams


def trajectory_inscene(cfg: Config, n_frames: int, first: int = 0, height: float = 6.0, ahead: float = 20.0,
                       drop: float = 3.0) -> list[CameraModel]:
    """SURVEY.md §8d's trajectory: a closed loop through the scene at `height` m (a circle
    of radius 0.3 side perturbed by a third harmonic), looking at a target `ahead` m
    along the path and `drop` m lower (pitched ~8.5 deg down); 1000 frames per loop.
    Near-plane, inside-box (granularity = inf) and far-LOD nodes all occur.  Under the
    reference's projection the city splats just in front of the image plane beside
    the camera become screen-covering ellipses (no frustum cull, render.hpp:104-156)
    that sort first and saturate every pixel: the frames exercise the cut, the
    preprocess and the sorts at full load, and the blend hardly at all."""
    side = scene_side(cfg.leaves)
    R, wob = 0.3 * side, 0.1 * side

    def at(a):
        return np.array([R * math.cos(a) + wob * math.sin(3 * a), height, R * math.sin(a)], np.float64)

    cams = []
    for i in range(first, first + n_frames):
        a = 2.0 * math.pi * (i % 1000) / 1000.0
        p = at(a)
        d = at(a + 1e-3) - p
        d[1] = 0.0
        d /= np.linalg.norm(d)
        target = p + ahead * d
        target[1] = height - drop
        cams.append(look_at_camera(p.astype(np.float32), target.astype(np.float32), cfg.width, cfg.height,
                                   cfg.focal))
    return cams


def camera(cfg: Config, frame: int = 0) -> CameraModel:
    return trajectory(cfg, 1, frame)[0]


def hierarchy(cfg: Config, seed: int = 1, threads: int = 0):
    return synth_city(cfg.leaves, seed=seed, threads=threads)


def chunk_parts(leaves: int, grid: int = 4, sky: int = 100_000, seed: int = 1):
    """The parts of a multi-chunk scene: grid x grid city chunks
    of leaves / grid^2 leaves each, tiled edge to edge around the origin, then a
    make_skybox shell (scene.hpp:111-137) 5 scene diameters out.  Yields
    (name, host Hierarchy) one part at a time so the caller can upload and free."""
    per = leaves // (grid * grid)
    side = scene_side(per)
    for iz in range(grid):
        for ix in range(grid):
            cx, cz = (ix - 0.5 * (grid - 1)) * side, (iz - 0.5 * (grid - 1)) * side
            yield f"chunk_{ix}_{iz}", synth_city_chunk(per, seed * 1009 + iz * grid + ix, cx, cz)
    if sky:
        yield "skybox", synth_skybox(sky, grid * side * math.sqrt(2.0), seed)


def multichunk(renderer, leaves: int, grid: int = 4, sky: int = 100_000, seed: int = 1, validate: bool = False):
    """Generate the chunks + skybox, upload each, and consolidate them on the device
    (hs_hierarchy_assemble: one merged root, breadth-first layout).  The parts are
    released once assembled; only the consolidated hierarchy stays resident."""
    parts = []
    for _, h in chunk_parts(leaves, grid, sky, seed):
        parts.append(renderer.upload(h, validate=validate))
        del h
    dh = renderer.assemble(parts)
    del parts
    return dh
