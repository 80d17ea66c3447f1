"""Multi-rank trajectory replay: the frame partition, the
per-frame image gather to rank 0 and the stats all_gather must reproduce the
single-rank replay exactly — same cut sizes, transferred counts, duplicates and
bit-identical images per frame.

CPU tests: gloo, world_size 2, with the CPU oracle as the frame source (test
infrastructure).  GPU test: two processes sharing one GPU, each with its own
Renderer (the product path, multi.GpuFrameSource), gathered over gloo with
host tensors — the same ImageGather code that runs over NCCL with device
tensors on a multi-GPU node."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2406_12080_b200 import multi

EXACT_COLS = ("rendered", "rendered_pct", "transferred", "n_duplicates")


def test_partition_even_blocks():
    for n in (1, 2, 7, 10, 1000):
        for world in (1, 2, 3, 4, 8):
            spans = [multi.partition(n, world, r) for r in range(world)]
            covered = [i for a, b in spans for i in range(a, b)]
            assert covered == list(range(n))
            for a, b in spans:
                assert b == a or a % 2 == 0  # refresh pairs never straddle ranks


class OracleSource(multi.FrameSource):
    def __init__(self, h):
        from oracle import oracle as orc
        self.orc = orc
        self.oh = orc.OracleHierarchy(h)
        self.cut = None
        self.prev = np.empty(0, np.uint32)
        self.last = None

    def _refresh(self, cam, tau):
        node, t, a = self.orc.select_cut(self.oh, cam, tau)
        self.cut = (node, t, a)
        fresh = int(np.count_nonzero(~np.isin(node, self.prev, assume_unique=True)))
        self.prev = node
        return fresh

    def prime(self, cam, tau):
        self._refresh(cam, tau)

    def frame(self, cam, tau, refreshed):
        d = {k: 0.0 for k in ("cut_expand", "weights", "preprocess", "duplicate", "tile_ranges", "alpha_blend")}
        if refreshed:
            d["transferred"] = self._refresh(cam, tau)
        sp = self.orc.cut_render_splats(self.oh, *self.cut)
        f = self.orc.render_forward(sp, cam)
        self.last = f
        d["n_duplicates"] = f.sizes()["n_entries"]
        d["rendered"] = len(self.cut[0])
        return d

    def image_into(self, buf):
        c, dep, T, _ = self.last.images()
        buf.copy_(torch.from_numpy(np.concatenate([c.ravel(), dep.ravel(), T.ravel()])))

    def leaf_count(self):
        return self.oh.leaf_count()


def _scene(n_frames=10):
    from paper_2406_12080_b200 import scenes
    cfg = scenes.Config("t", 3000, 96, 64, 60.0, 3.0, altitude=8.0, standoff=5.0, lookahead=20.0)
    import paper_2406_12080_b200 as hs
    h = hs.synth_city(cfg.leaves, seed=11)
    return h, scenes.trajectory(cfg, n_frames, first=100), cfg.tau


def _collect(store):
    def on_image(i, t):
        store[i] = t.detach().cpu().numpy().view(np.uint32).copy()
    return on_image


def _worker(rank, world, port, q, n_frames):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h, cams, tau = _scene(n_frames)
    imgs = {}
    stats = multi.replay_trajectory(OracleSource(h), cams, tau, gather_images=True, on_image=_collect(imgs))
    if rank == 0:
        q.put((stats, imgs))
    else:
        assert not imgs  # images land on rank 0 only
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return got


@pytest.mark.parametrize("world,n_frames", [(2, 10), (3, 9)])
def test_multi_rank_replay_matches_single_rank(world, n_frames):
    """Stats and every frame's image gathered to rank 0 equal the 1-rank replay
    bit for bit (9 frames over 3 ranks: blocks of 4, 4, 1 — a short last block)."""
    h, cams, tau = _scene(n_frames)
    single_imgs = {}
    single = multi.replay_trajectory(OracleSource(h), cams, tau, gather_images=True,
                                     on_image=_collect(single_imgs))
    got, imgs = _spawn(_worker, world, n_frames)
    cols = [multi.STAT_FIELDS.index(k) for k in EXACT_COLS]
    assert np.array_equal(got[:, cols], single[:, cols])
    assert got[0, multi.STAT_FIELDS.index("transferred")] == got[0, 0]  # frame 0 uploads its whole cut
    assert np.all(got[1::2, multi.STAT_FIELDS.index("transferred")] == 0)
    assert sorted(imgs) == list(range(n_frames))
    for i in range(n_frames):
        assert np.array_equal(imgs[i], single_imgs[i]), f"frame {i}"


def _gpu_worker(rank, world, port, q, n_frames):
    import torch.distributed as dist

    import paper_2406_12080_b200 as hs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h, cams, tau = _scene(n_frames)
    r = hs.Renderer(0)
    imgs = {}
    stats = multi.replay_trajectory(multi.GpuFrameSource(r, r.upload(h)), cams, tau, device="cpu",
                                    gather_images=True, on_image=_collect(imgs))
    if rank == 0:
        q.put((stats, imgs))
    dist.barrier()
    r.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_gpu_replay_matches_single_rank():
    """The product path on two ranks (two processes sharing the GPU): per-frame
    images and stats bitwise equal to the single-rank GPU replay, which itself
    equals the oracle frame for frame."""
    import paper_2406_12080_b200 as hs
    n_frames = 10
    h, cams, tau = _scene(n_frames)
    r = hs.Renderer(0)
    single_imgs = {}
    single = multi.replay_trajectory(multi.GpuFrameSource(r, r.upload(h)), cams, tau, gather_images=True,
                                     on_image=_collect(single_imgs))
    r.close()
    oracle_imgs = {}
    oracle = multi.replay_trajectory(OracleSource(h), cams, tau, gather_images=True, on_image=_collect(oracle_imgs))
    got, imgs = _spawn(_gpu_worker, 2, n_frames)
    cols = [multi.STAT_FIELDS.index(k) for k in EXACT_COLS]
    assert np.array_equal(got[:, cols], single[:, cols])
    assert np.array_equal(single[:, cols], oracle[:, cols])
    for i in range(n_frames):
        assert np.array_equal(imgs[i], single_imgs[i]), f"frame {i}"
        assert np.array_equal(imgs[i], oracle_imgs[i]), f"frame {i} vs oracle"
    # refresh frames carry a timed cut (bench_path times select_cut), odd frames none
    ce = multi.STAT_FIELDS.index("cut_expand")
    assert np.all(single[0::2, ce] > 0) and np.all(single[1::2, ce] == 0)
