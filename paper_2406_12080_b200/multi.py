"""View-parallel trajectory replay across GPUs.

The hierarchy is replicated on every rank; a camera trajectory's frames are
split into contiguous, even-length blocks so that the reference cadence of
bench_path (bench.hpp:55-103: cut refreshed on even frames, reused on odd
ones) never straddles two ranks.  A rank r > 0 also selects the cut of the
refresh frame just before its block (`FrameSource.prime`), so its first
frame's `transferred` statistic (new cut nodes vs the previous refresh) equals
the single-GPU value.

Frames need no exchange while rendering.  The data plane is the gather the
north star reserves NCCL for:
  * per-frame images go to rank 0 while the ranks keep rendering: after frame
    k of its block, every rank r > 0 posts an asynchronous send of its image
    (colour, inverse depth, transmittance planes; 20 B/pixel) and rank 0 posts
    the matching receives (`batch_isend_irecv`: one grouped NCCL launch per
    step over NVLink), double-buffered so frame k's transfer overlaps frame
    k+1's kernels;
  * the fixed-size per-frame stats are gathered once at the end (all_gather).
On GPU ranks the images move device to device (hs_frame_download_device into
a tensor NCCL sends); the CPU tests run the same code over gloo with host
tensors.
"""
from __future__ import annotations

import numpy as np

STAT_FIELDS = ("rendered", "rendered_pct", "transferred", "cut_expand", "weights", "preprocess", "duplicate",
               "tile_ranges", "alpha_blend", "n_duplicates")
PLANES = 5  # colour (3), inverse depth, transmittance (RenderOutput, render.hpp:77-83)


def partition(n_frames: int, world: int, rank: int) -> tuple[int, int]:
    """Frames [start, stop) of `rank`: blocks of B = 2 * ceil(F / (2 G)) frames."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    block = 2 * -(-n_frames // (2 * world))
    start = min(n_frames, rank * block)
    return start, min(n_frames, start + block)


class FrameSource:
    """What a rank needs to replay frames (the bench_path loop body, bench.hpp:70-97).

    prime(cam, tau): select the cut of the refresh frame before the rank's block
        and count it in the transfer tracker (not a frame of this rank: no stats).
    frame(cam, tau, refreshed) -> dict: render one frame, refreshing the cut on
        even frames; returns the cut size ("rendered"), "transferred" (refresh
        frames), the six stage times in seconds and "n_duplicates".
    image_into(buf): write the last frame's planes (PLANES, H, W) float32 into
        `buf` (a torch tensor on the rank's device or on the host).
    """

    def prime(self, cam, tau) -> None:  # pragma: no cover - interface
        raise NotImplementedError

    def frame(self, cam, tau, refreshed: bool) -> dict:  # pragma: no cover - interface
        raise NotImplementedError

    def image_into(self, buf) -> None:  # pragma: no cover - interface
        raise NotImplementedError

    def leaf_count(self) -> int:  # pragma: no cover - interface
        raise NotImplementedError


class GpuFrameSource(FrameSource):
    """FrameSource over a Renderer + device hierarchy (the product path): refresh
    frames are render_hierarchy with per-stage CUDA events (the cut is timed, as
    in bench_path), odd frames render the previous cut; cut churn is counted on
    the device."""

    def __init__(self, renderer, dh):
        from . import _native as N
        self.N = N
        self.L = N.lib()
        self.r = renderer
        self.dh = renderer._dev(dh)
        self.tracker = renderer.transfer_tracker(self.dh)
        self.cut_size = 0

    def _check(self, status):
        from . import _check
        _check(status, self.r.ctx)

    def prime(self, cam, tau):
        self.cut_size = self.r.select_cut_device(self.dh, cam, tau)
        self.tracker.count(self.r._cut)

    def frame(self, cam, tau, refreshed):
        N, L, r = self.N, self.L, self.r
        st = N.hs_stage_times()
        cc = cam.to_c()
        out = {}
        if refreshed:
            self._check(L.hs_render_hierarchy(r.ctx, self.dh.handle, N.C.byref(cc), float(tau), r._cut, r._frame,
                                              N.C.byref(st)))
            n = N.C.c_uint64()
            self._check(L.hs_cut_size(r.ctx, r._cut, N.C.byref(n)))
            self.cut_size = int(n.value)
            out["transferred"] = self.tracker.count(r._cut)
        else:
            self._check(L.hs_render_cut(r.ctx, self.dh.handle, r._cut, N.C.byref(cc), r._frame, N.C.byref(st)))
        fi = N.hs_frame_info()
        self._check(L.hs_frame_get_info(r.ctx, r._frame, N.C.byref(fi)))
        for k in ("cut_expand", "weights", "preprocess", "duplicate", "tile_ranges", "alpha_blend"):
            out[k] = getattr(st, k)
        out["rendered"] = self.cut_size
        out["n_duplicates"] = int(fi.n_duplicates)
        self.wh = (int(fi.width), int(fi.height))
        return out

    def image_into(self, buf):
        import torch
        N, L, r = self.N, self.L, self.r
        W, H = self.wh
        assert buf.dtype == torch.float32 and buf.is_contiguous() and buf.numel() == PLANES * W * H
        f32 = N.C.POINTER(N.C.c_float)
        p = buf.data_ptr()
        col, dep, tr = (N.C.cast(p, f32), N.C.cast(p + 12 * W * H, f32), N.C.cast(p + 16 * W * H, f32))
        if buf.is_cuda:  # device to device on the caller's (torch) stream: NCCL reads it from there
            s = torch.cuda.current_stream(buf.device).cuda_stream
            self._check(L.hs_frame_download_device(r.ctx, r._frame, col, dep, tr, N.C.c_void_p(s)))
        else:
            rc = N.C.c_int32()
            self._check(L.hs_frame_download(r.ctx, r._frame, col, dep, tr, N.C.byref(rc)))

    def leaf_count(self):
        return self.dh.leaf_count()


def _row(st: dict, refreshed: bool, leaves: int) -> list[float]:
    row = dict.fromkeys(STAT_FIELDS, 0.0)
    for k, v in st.items():
        if k in row:
            row[k] = float(v)
    if not refreshed:  # odd frames cost no cut work and move nothing (bench.hpp:70-84)
        row["cut_expand"] = row["weights"] = row["transferred"] = 0.0
    row["rendered_pct"] = 100.0 * row["rendered"] / leaves
    return [row[k] for k in STAT_FIELDS]


def replay_block(src: FrameSource, cams, tau: float, start: int, stop: int, on_frame=None) -> np.ndarray:
    """bench_path (bench.hpp:55-103) over frames [start, stop) of `cams`; returns a
    (stop-start, len(STAT_FIELDS)) float64 array.  on_frame(i) runs after frame i."""
    leaves = src.leaf_count()
    out = np.zeros((stop - start, len(STAT_FIELDS)), np.float64)
    if start > 0:  # the previous refresh, for the transferred statistic
        src.prime(cams[start - 2 if start >= 2 else 0], tau)
    for i in range(start, stop):
        refreshed = i % 2 == 0
        out[i - start] = _row(src.frame(cams[i], tau, refreshed), refreshed, leaves)
        if on_frame is not None:
            on_frame(i)
    return out


class ImageGather:
    """Per-frame images of every rank to rank 0, overlapped with rendering.

    Step k (the k-th frame of every rank's block): rank r > 0 copies its image
    into send slot k % 2 and posts the send; rank 0 posts receives for every
    rank that has a k-th frame into recv slot k % 2.  Slot k % 2 is reused at
    step k + 2 only after the step-k transfers completed, so each transfer
    overlaps the next frame's kernels.  Rank 0 hands every image, in trajectory
    order per rank, to on_image(frame_index, tensor) once it has landed.
    """

    def __init__(self, src: FrameSource, n_frames: int, shape, group=None, device=None, on_image=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.src, self.group = src, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.spans = [partition(n_frames, self.world, r) for r in range(self.world)]
        self.on_image = on_image
        self.device = device
        self.bytes_moved = 0
        mk = lambda: torch.empty(PLANES * shape[0] * shape[1], dtype=torch.float32, device=device)  # noqa: E731
        if self.rank == 0:
            self.own = mk()
            self.recv = {r: [mk(), mk()] for r in range(1, self.world)}
        else:
            self.send = [mk(), mk()]
        self.works = [[], []]
        self.landed = [[], []]  # (frame index, tensor) delivered when the slot's works finish

    def _finish(self, slot: int):
        for w in self.works[slot]:
            w.wait()
        self.works[slot] = []
        for i, t in self.landed[slot]:
            if self.on_image is not None:
                self.on_image(i, t)
        self.landed[slot] = []

    def step(self, k: int):
        """After every rank rendered (or skipped) the k-th frame of its block."""
        dist = self.dist
        slot = k % 2
        self._finish(slot)  # step k - 2's transfers: the slot is free again
        ops = []
        if self.rank == 0:
            s0, e0 = self.spans[0]
            if k < e0 - s0:
                self.src.image_into(self.own)
                if self.on_image is not None:
                    self.on_image(s0 + k, self.own)
            for r in range(1, self.world):
                s, e = self.spans[r]
                if k < e - s:
                    buf = self.recv[r][slot]
                    ops.append(dist.P2POp(dist.irecv, buf, r, self.group))
                    self.landed[slot].append((s + k, buf))
                    self.bytes_moved += buf.numel() * 4
        else:
            s, e = self.spans[self.rank]
            if k < e - s:
                buf = self.send[slot]
                self.src.image_into(buf)
                ops.append(dist.P2POp(dist.isend, buf, 0, self.group))
                self.bytes_moved += buf.numel() * 4
        if ops:
            self.works[slot] = dist.batch_isend_irecv(ops)

    def close(self):
        self._finish(0)
        self._finish(1)


def replay_trajectory(src: FrameSource, cams, tau: float, group=None, device=None, gather_images: bool = False,
                      on_image=None) -> np.ndarray:
    """Replay the whole trajectory across the ranks of `group` (or locally when
    torch.distributed is not initialised); every rank returns all frames' stats.
    With gather_images, rank 0 receives every frame's image (on_image(i, tensor)
    per frame, in each rank's frame order) while the ranks render."""
    import torch
    import torch.distributed as dist

    n = len(cams)
    if device is None:
        device = "cuda" if (dist.is_available() and dist.is_initialized()
                            and dist.get_backend(group) == "nccl") else "cpu"
    if not (dist.is_available() and dist.is_initialized()):
        buf = None

        def local_frame(i):
            nonlocal buf
            if gather_images and on_image is not None:
                if buf is None:
                    W, H = cams[i].width, cams[i].height
                    buf = torch.empty(PLANES * W * H, dtype=torch.float32, device=device)
                src.image_into(buf)
                on_image(i, buf)
        return replay_block(src, cams, tau, 0, n, on_frame=local_frame)

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    start, stop = partition(n, world, rank)
    block = 2 * -(-n // (2 * world))
    gather = None
    if gather_images:
        gather = ImageGather(src, n, (cams[0].height, cams[0].width), group, device, on_image)
    local = np.zeros((block, len(STAT_FIELDS)), np.float64)
    if stop > start:
        local[: stop - start] = replay_block(src, cams, tau, start, stop,
                                             on_frame=(lambda i: gather.step(i - start)) if gather else None)
    if gather is not None:
        for k in range(stop - start, block):  # steps this rank has no frame for (a shorter last block)
            gather.step(k)
        gather.close()
    t = torch.from_numpy(local).to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    full = torch.cat(parts).cpu().numpy()
    return full[:n]
