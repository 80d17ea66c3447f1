"""View-parallel trajectory replay across GPUs.

The hierarchy is replicated on every rank; a camera trajectory's frames are
split into contiguous, even-length blocks so that the reference cadence of
bench_path (bench.hpp:55-103: cut refreshed on even frames, reused on odd
ones) never straddles two ranks.  A rank r > 0 also selects the cut of the
refresh frame just before its block, so its first frame's `transferred`
statistic (new cut nodes vs the previous refresh) equals the single-GPU
value.  Frames need no exchange while rendering; the per-frame statistics are
gathered once at the end with one all_gather (NCCL over NVLink for GPU ranks,
gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np

STAT_FIELDS = ("rendered", "rendered_pct", "transferred", "cut_expand", "weights", "preprocess", "duplicate",
               "tile_ranges", "alpha_blend", "n_duplicates")


def partition(n_frames: int, world: int, rank: int) -> tuple[int, int]:
    """Frames [start, stop) of `rank`: blocks of B = 2 * ceil(F / (2 G)) frames."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    block = 2 * -(-n_frames // (2 * world))
    start = min(n_frames, rank * block)
    return start, min(n_frames, start + block)


class FrameSource:
    """What a rank needs to replay frames: `refresh(cam, tau) -> (cut size,
    transferred)` selects a new cut and counts its nodes absent from the
    previous refresh (bench.hpp:79-82), and `render(cam) -> dict of stage
    seconds (+ n_duplicates)` renders the last cut."""

    def refresh(self, cam, tau) -> tuple[int, int]:  # pragma: no cover - interface
        raise NotImplementedError

    def render(self, cam, refreshed: bool) -> dict:  # pragma: no cover - interface
        raise NotImplementedError

    def leaf_count(self) -> int:  # pragma: no cover - interface
        raise NotImplementedError


class GpuFrameSource(FrameSource):
    """FrameSource over a Renderer + device hierarchy (the product path)."""

    def __init__(self, renderer, dh):
        self.r = renderer
        self.dh = dh
        self.tracker = renderer.transfer_tracker(dh)  # cut churn counted on the device

    def refresh(self, cam, tau):
        n = self.r.select_cut_device(self.dh, cam, tau)
        return n, self.tracker.count(self.r._cut)

    def render(self, cam, refreshed):
        from . import StageTimes
        st = StageTimes()
        out = self.r.render_cut(self.dh, cam, stages=st)
        d = dict(vars(st))
        d["n_duplicates"] = out.info["n_duplicates"]
        return d

    def leaf_count(self):
        return self.dh.leaf_count()


def replay_block(src: FrameSource, cams, tau: float, start: int, stop: int) -> np.ndarray:
    """bench_path (bench.hpp:55-103) over frames [start, stop) of `cams`; returns
    a (stop-start, len(STAT_FIELDS)) float64 array."""
    leaves = src.leaf_count()
    out = np.zeros((stop - start, len(STAT_FIELDS)), np.float64)
    cut_size = 0
    if start > 0:  # the previous refresh, for the transferred statistic
        cut_size, _ = src.refresh(cams[start - 2 if start >= 2 else 0], tau)
    for i in range(start, stop):
        refreshed = i % 2 == 0
        row = dict.fromkeys(STAT_FIELDS, 0.0)
        if refreshed:
            cut_size, transferred = src.refresh(cams[i], tau)
            row["transferred"] = float(transferred)
        st = src.render(cams[i], refreshed)
        for k, v in st.items():
            if k in row and k not in ("rendered", "rendered_pct", "transferred"):
                row[k] = float(v)
        if not refreshed:
            row["cut_expand"] = 0.0
            row["weights"] = 0.0
        row["rendered"] = float(cut_size)
        row["rendered_pct"] = 100.0 * cut_size / leaves
        out[i - start] = [row[k] for k in STAT_FIELDS]
    return out


def replay_trajectory(src: FrameSource, cams, tau: float, group=None, device=None) -> np.ndarray:
    """Replay the whole trajectory across the ranks of `group` (or locally when
    torch.distributed is not initialised); every rank returns all frames' stats."""
    import torch
    import torch.distributed as dist

    n = len(cams)
    if not (dist.is_available() and dist.is_initialized()):
        return replay_block(src, cams, tau, 0, n)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    start, stop = partition(n, world, rank)
    block = 2 * -(-n // (2 * world))
    local = np.zeros((block, len(STAT_FIELDS)), np.float64)
    if stop > start:
        local[: stop - start] = replay_block(src, cams, tau, start, stop)
    if device is None:
        device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.from_numpy(local).to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    full = torch.cat(parts).cpu().numpy()
    return full[:n]
