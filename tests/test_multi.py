"""Multi-rank trajectory replay on CPU (gloo, world_size 2): the frame
partition and the stats gather must reproduce the single-rank replay exactly
(same cut sizes, transferred counts and duplicates per frame).  The frame
source here is the CPU oracle (test infrastructure); on GPUs it is the
Renderer (multi.GpuFrameSource)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2406_12080_b200 import multi


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

    def refresh(self, cam, tau):
        node, t, a = self.orc.select_cut(self.oh, cam, tau)
        self.cut = (node, t, a)
        fresh = int(np.count_nonzero(~np.isin(node, self.prev, assume_unique=True)))
        self.prev = node
        return len(node), fresh

    def render(self, cam, refreshed):
        sp = self.orc.cut_render_splats(self.oh, *self.cut)
        f = self.orc.render_forward(sp, cam)
        d = {k: 0.0 for k in ("cut_expand", "weights", "preprocess", "duplicate", "tile_ranges", "alpha_blend")}
        d["n_duplicates"] = f.sizes()["n_entries"]
        return d

    def leaf_count(self):
        return self.oh.leaf_count()


def _scene():
    from paper_2406_12080_b200 import scenes
    cfg = scenes.Config("t", 3000, 96, 64, 60.0, 3.0, altitude=8.0, standoff=5.0, lookahead=20.0)
    import paper_2406_12080_b200 as hs
    h = hs.synth_city(cfg.leaves, seed=11)
    return h, scenes.trajectory(cfg, 10, first=100), cfg.tau


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h, cams, tau = _scene()
    stats = multi.replay_trajectory(OracleSource(h), cams, tau)
    if rank == 0:
        q.put(stats)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_replay_matches_single_rank():
    h, cams, tau = _scene()
    single = multi.replay_trajectory(OracleSource(h), cams, tau)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cols = [multi.STAT_FIELDS.index(k) for k in ("rendered", "rendered_pct", "transferred", "n_duplicates")]
    assert np.array_equal(got[:, cols], single[:, cols])
    assert got[0, multi.STAT_FIELDS.index("transferred")] == got[0, 0]  # frame 0 uploads its whole cut
    assert np.all(got[1::2, multi.STAT_FIELDS.index("transferred")] == 0)
