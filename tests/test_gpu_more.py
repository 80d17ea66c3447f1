"""More GPU parity: full-size BASELINE config (C2, 10M leaves, 1080p) against
the oracle, bench_path cadence/transfer accounting, capacity growth, .h3dg
loading on the device, degenerate hierarchies and the fast blend mode's
tolerance.  All through the C ABI."""
import numpy as np
import pytest

import paper_2406_12080_b200 as hs
from oracle import oracle as orc
from paper_2406_12080_b200 import multi, scenes
from tests.fixtures import Rng, axis_camera, gray_splat, random_gaussians

pytestmark = pytest.mark.gpu


def images_equal(out, f):
    c, d, t, rc = f.images()
    return (np.array_equal(out.color.view(np.uint32), c.view(np.uint32))
            and np.array_equal(out.depth.view(np.uint32), d.view(np.uint32))
            and np.array_equal(out.transmittance.view(np.uint32), t.view(np.uint32)) and out.rendered_count == rc)


def test_c2_full_size_bit_exact(renderer, c2, c2_oracle, c2_device):
    """BASELINE config[1]: cut, sorted keys/tile ranges and image bit-exact vs the oracle."""
    cfg, h = c2
    cam = scenes.camera(cfg, 100)
    dh = c2_device
    out, cut = renderer.render_hierarchy(dh, cam, cfg.tau, want_context=True, return_cut=True)
    f = orc.render_hierarchy(c2_oracle, cam, cfg.tau, keep_ctx=True)
    node, t, a = f.cut()
    assert np.array_equal(cut.node, node)
    assert np.array_equal(cut.t.view(np.uint32), t.view(np.uint32))
    assert np.array_equal(cut.alpha_prime.view(np.uint32), a.view(np.uint32))
    oc = f.context()
    assert np.array_equal(out.context["tile_start"], oc["tile_start"])
    assert np.array_equal(out.context["sorted_vals"], oc["tile_entries"])
    keys = out.context["sorted_keys"]
    assert np.all(keys[1:] >= keys[:-1])  # sortedness at full size
    assert images_equal(out, f)
    # cut partitions the leaves (test_lod.cpp:176-199): no selected node has a selected
    # parent, and the selected subtrees' leaf counts add up to all leaves
    sel = np.zeros(h.n, bool)
    sel[cut.node] = True
    par = h.parent[cut.node]
    assert not np.any(sel[par[par != hs.NO_NODE]])
    # leaves under each node, accumulated bottom-up level by level (parent < child)
    depth = np.zeros(h.n, np.int32)
    for lvl in range(64):  # propagate depth: parent depth + 1 (converges in tree height)
        nd = np.where(h.parent == hs.NO_NODE, 0, depth[np.where(h.parent == hs.NO_NODE, 0, h.parent)] + 1)
        if np.array_equal(nd, depth):
            break
        depth = nd.astype(np.int32)
    under = (h.child_count == 0).astype(np.int64)
    for lvl in range(int(depth.max()), 0, -1):
        idx = np.flatnonzero(depth == lvl)
        np.add.at(under, h.parent[idx], under[idx])
    assert int(under[cut.node].sum()) == h.leaf_count()


def test_c2_fast_mode_within_tolerance(c2, c2_oracle):
    cfg, h = c2
    cam = scenes.camera(cfg, 333)
    r = hs.Renderer(0, exact=False)
    out = r.render_hierarchy(h, cam, cfg.tau)
    f = orc.render_hierarchy(c2_oracle, cam, cfg.tau, keep_ctx=False)
    c, d, t, rc = f.images()
    assert np.abs(out.color - c).max() <= 1e-3
    assert np.abs(out.transmittance - t).max() <= 1e-3
    assert hs.psnr(out.color, c) >= 50.0
    r.close()


def test_bench_path_matches_oracle(renderer):
    rng = Rng(22)
    h = hs.build_bvh(*random_gaussians(rng, 400, 4.0, 0.05, 0.2, 0.3, 0.9))
    cams = [hs.look_at_camera([0, 0, z], [0, 0, 0], 64, 48, 60.0) for z in (-40, -40, -12, -12, -3.5, -3.5, -30)]
    rep = hs.bench_path(h, cams, 4.0, renderer=renderer)
    st = orc.bench_path(orc.OracleHierarchy(h), cams, 4.0)
    assert [f.rendered for f in rep.frames] == list(st[:, 0].astype(int))
    assert [f.transferred for f in rep.frames] == list(st[:, 2].astype(int))
    assert all(f.stages.cut_expand == 0 for f in rep.frames[1::2])
    lines = rep.csv().strip().split("\n")
    assert lines[0].startswith("frame,rendered,rendered_pct,transferred,cut_expand_s")
    assert len(lines) == len(cams) + 2 and lines[-1].startswith("total,")


def test_trajectory_replay_single_gpu_matches_bench_path(renderer):
    cfg = scenes.CONFIGS["c1"]
    h = scenes.hierarchy(cfg)
    dh = renderer.upload(h)
    cams = scenes.trajectory(cfg, 8, first=40)
    stats = multi.replay_trajectory(multi.GpuFrameSource(renderer, dh), cams, cfg.tau)
    rep = hs.bench_path(dh, cams, cfg.tau, renderer=renderer)
    assert list(stats[:, 0].astype(int)) == [f.rendered for f in rep.frames]
    assert list(stats[:, 2].astype(int)) == [f.transferred for f in rep.frames]


def test_transfer_tracker_matches_set_difference(renderer):
    """hs_transfer_count == |cut \\ previous cut| (bench.hpp:79-82) over a trajectory
    with churn, a repeated cut (0 new) and a tau jump (large churn)."""
    cfg = scenes.CONFIGS["c1"]
    h = scenes.hierarchy(cfg)
    dh = renderer.upload(h)
    tr = renderer.transfer_tracker(dh)
    cams = scenes.trajectory(cfg, 6, first=300)
    steps = [(c, cfg.tau) for c in cams] + [(cams[-1], cfg.tau), (cams[-1], 12.0), (cams[0], 0.0)]
    prev = np.empty(0, np.uint32)
    for cam, tau in steps:
        cut = renderer.select_cut(dh, cam, tau)
        want = int(np.count_nonzero(~np.isin(cut.node, prev, assume_unique=True)))
        assert tr.count() == want
        prev = cut.node
    other = renderer.upload(scenes.hierarchy(scenes.Config("o", 500, 64, 48, 60.0, 3.0)))
    with pytest.raises(hs.Error):
        renderer.transfer_tracker(other).count()  # the current cut belongs to `dh`
    tr.close()


def test_duplicate_buffer_grows(renderer):
    """Splats covering every tile overflow the initial key buffer; the synchronous
    call grows it and re-runs (results still bit-exact)."""
    cam = axis_camera(1024, 1024, 40.0)
    parts = [gray_splat([0.01 * i, 0, 0.6], 2.5, 0.05) for i in range(400)]
    from tests.fixtures import concat
    sp = concat(parts)
    r = hs.Renderer(0, exact=True)
    out = r.render_forward(sp, cam)
    assert out.info["n_duplicates"] > 4 * len(sp)
    f = orc.render_forward(sp, cam, keep_ctx=False)
    assert images_equal(out, f)
    r.close()


def test_load_h3dg_on_device(renderer, tmp_path):
    h = hs.synth_city(3000, seed=5)
    p = str(tmp_path / "x.h3dg")
    hs.write_hierarchy(p, h)
    dh = renderer.load_h3dg(p)
    assert dh.n == h.n and dh.leaf_count() == h.leaf_count()
    cam = hs.look_at_camera([0, 10, -40], [0, 0, 0], 96, 64, 80.0)
    a = renderer.render_hierarchy(dh, cam, 3.0)
    b = renderer.render_hierarchy(h, cam, 3.0)
    assert np.array_equal(a.color.view(np.uint32), b.color.view(np.uint32))
    bad = tmp_path / "bad.h3dg"
    bad.write_bytes(open(p, "rb").read()[:-3])
    with pytest.raises(hs.Error) as e:
        renderer.load_h3dg(str(bad))
    assert e.value.code == hs.Errc.TruncatedRecord


def test_single_node_and_camera_inside_root(renderer):
    rng = Rng(3)
    m, s, q, f, sh = random_gaussians(rng, 1, 1.0, 0.2, 0.4, 0.5, 0.9)
    h = hs.build_bvh(m, s, q, f, sh)  # one leaf = the root
    cam = hs.look_at_camera([0, 0, -6], [0, 0, 0], 48, 40, 60.0)
    cut = renderer.select_cut(h, cam, 3.0)
    assert list(cut.node) == [0] and cut.t[0] == 1.0
    h2 = hs.synth_city(2000, seed=8)
    inside = hs.look_at_camera([0, 2, 0], [0, 0, 30], 64, 48, 60.0)  # inside the root box: eps = inf
    out, cut2 = renderer.render_hierarchy(h2, inside, 3.0, return_cut=True)
    f = orc.render_hierarchy(orc.OracleHierarchy(h2), inside, 3.0, keep_ctx=False)
    assert np.array_equal(cut2.node, f.cut()[0])
    assert images_equal(out, f)


def test_tau_zero_renders_every_leaf(renderer):  # test_bench.cpp:115-128
    h = hs.synth_city(1500, seed=9)
    cam = hs.look_at_camera([0, 20, -60], [0, 0, 0], 80, 60, 70.0)
    out, cut = renderer.render_hierarchy(h, cam, 0.0, return_cut=True)
    assert np.array_equal(cut.node, np.flatnonzero(h.child_count == 0))
    assert np.all(cut.t == 1.0)
    f = orc.render_hierarchy(orc.OracleHierarchy(h), cam, 0.0, keep_ctx=False)
    assert images_equal(out, f)
