"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bit-exact for the cut (nodes, t, alpha'), the per-splat
projection (z, radius, rect), the duplicated and sorted key lists, the tile
ranges and rendered_count; images bit-exact in exact blend mode (the bar is
max-abs <= 1e-3 per channel and PSNR >= 50 dB, asserted separately for the
fast mode)."""
import numpy as np
import pytest

import paper_2406_12080_b200 as hs
from oracle import oracle as orc
from paper_2406_12080_b200 import scenes
from tests.fixtures import Rng, random_camera, random_hierarchy, random_scene, random_scene_camera

pytestmark = pytest.mark.gpu

MAX_ABS = 1e-3  # north_star: images within max-abs 1e-3 per channel
MIN_PSNR = 50.0


def oracle_keys(ctx_o, zbits):
    """ForwardContext (tile_start, tile_entries) expressed as the GPU's sorted key list."""
    ts = ctx_o["tile_start"].astype(np.int64)
    te = ctx_o["tile_entries"]
    tiles = np.repeat(np.arange(len(ts) - 1, dtype=np.uint64), np.diff(ts))
    return (tiles << np.uint64(32)) | zbits[te].astype(np.uint64), te


def zbits_of(proj16):
    return proj16[:, 1].view(np.uint32)


def assert_images(out, f, exact=True):
    c, d, t, rc = f.images()
    if exact:
        assert np.array_equal(out.color.view(np.uint32), c.view(np.uint32)), "color differs"
        assert np.array_equal(out.depth.view(np.uint32), d.view(np.uint32)), "depth differs"
        assert np.array_equal(out.transmittance.view(np.uint32), t.view(np.uint32)), "T differs"
    else:
        assert np.abs(out.color - c).max() <= MAX_ABS
        assert hs.psnr(out.color, c) >= MIN_PSNR
    assert out.rendered_count == rc


def check_forward_context(out, f):
    """Sorted keys / ids / tile_start bit-exact; duplicated (pre-sort) list bit-exact."""
    oc = f.context()
    gctx = out.context
    assert np.array_equal(gctx["tile_start"], oc["tile_start"])
    assert np.array_equal(gctx["sorted_vals"], oc["tile_entries"])
    # the GPU keys carry bits(cam z) of the splat; recompute from the oracle's dump
    keys_o, _ = oracle_keys(oc, zbits_of(oc["proj16"]))
    assert np.array_equal(gctx["sorted_keys"], keys_o)
    # pre-sort duplicate list: splat id asc, ty asc, tx asc (render.hpp:273-294 emission order)
    pj = oc["proj16"]
    vis = np.flatnonzero(pj[:, 0] == 0)
    tx0, ty0 = pj[:, 14].view(np.int32), pj[:, 15].view(np.int32)
    rect = pj[:, 13].view(np.uint32)
    tx1, ty1 = (rect >> 8) & 0xFF, (rect >> 24) & 0xFF
    exp_k, exp_v = [], []
    tiles_x = oc["tiles_x"]
    zb = zbits_of(pj)
    for i in vis:
        for ty in range(ty0[i], ty1[i]):
            for tx in range(tx0[i], tx1[i]):
                exp_k.append((np.uint64(ty * tiles_x + tx) << np.uint64(32)) | np.uint64(zb[i]))
                exp_v.append(i)
    # the device emits the pairs in depth order (before the tile sort); compare as a multiset
    got = np.lexsort((gctx["dup_vals"], gctx["dup_keys"]))
    exp_k = np.array(exp_k, np.uint64)
    exp_v = np.array(exp_v, np.uint32)
    want = np.lexsort((exp_v, exp_k))
    assert np.array_equal(gctx["dup_keys"][got], exp_k[want])
    assert np.array_equal(gctx["dup_vals"][got], exp_v[want])


def check_projection(out, f):
    gp = out.context["proj16"]
    op = f.context()["proj16"]
    assert gp.shape == op.shape
    culled = op[:, 0] != 0
    assert np.array_equal(gp[:, 0] != 0, culled)
    v = ~culled
    # z, mean2d, conic, alpha_scale, colour, inv_depth, radius, rect: bit-exact
    assert np.array_equal(gp[v].view(np.uint32), op[v].view(np.uint32))


# ----------------------------------------------------------------------------- cut
@pytest.mark.parametrize("seed", range(6))
def test_cut_matches_oracle_random_trees(renderer, seed):
    rng = Rng(100 + seed)
    for _ in range(10):
        h = random_hierarchy(rng, 1 + rng.randint(300))
        cam = random_camera(rng, 5.0)
        tau = float(rng.uniform(0.5, 400.0))
        node, t, a = orc.select_cut(orc.OracleHierarchy(h), cam, tau)
        cut = renderer.select_cut(h, cam, tau)
        assert np.array_equal(cut.node, node)
        assert np.array_equal(cut.t.view(np.uint32), t.view(np.uint32))
        assert np.array_equal(cut.alpha_prime.view(np.uint32), a.view(np.uint32))


@pytest.mark.parametrize("tau", [0.0, 1.5, 3.0, 6.0, 12.0, 1e9])
def test_cut_tau_sweep_c1(renderer, c1, tau):
    h, oh, cam = c1
    node, t, a = orc.select_cut(oh, cam, tau)
    cut = renderer.select_cut(h, cam, tau)
    assert len(cut) == len(node)
    assert np.array_equal(cut.node, node)
    assert np.array_equal(cut.t.view(np.uint32), t.view(np.uint32))
    assert np.array_equal(cut.alpha_prime.view(np.uint32), a.view(np.uint32))


def test_cut_tau_on_node_granularities(renderer, c1):
    """k_select_cut compares RN(num / den) with tau without dividing (GranCmp): tau set
    to nodes' own granularities and their float neighbours (the comparisons' edges),
    denormal and extreme taus, all bit-exact against the oracle's divisions."""
    h, oh, cam = c1
    eps = renderer.granularity(h.bmin, h.bmax, cam)
    fin = np.flatnonzero(np.isfinite(eps) & (eps > 0))
    pick = eps[fin[np.linspace(0, len(fin) - 1, 5).astype(int)]]
    f32 = np.float32
    taus = [float(np.median(eps[fin]))]
    for e in pick:
        taus += [float(e), float(np.nextafter(f32(e), f32(np.inf))), float(np.nextafter(f32(e), f32(0)))]
    taus += [float(np.finfo(np.float32).smallest_subnormal), 1e-42, float(np.finfo(np.float32).max)]
    for tau in taus:
        node, t, a = orc.select_cut(oh, cam, tau)
        cut = renderer.select_cut(h, cam, tau)
        assert np.array_equal(cut.node, node), tau
        assert np.array_equal(cut.t.view(np.uint32), t.view(np.uint32)), tau
        assert np.array_equal(cut.alpha_prime.view(np.uint32), a.view(np.uint32)), tau


def test_cut_rejects_negative_tau(renderer, c1):
    h, _, cam = c1
    with pytest.raises(hs.Error) as e:
        renderer.select_cut(h, cam, -1.0)
    assert e.value.code == hs.Errc.InvalidArgument
    assert str(e.value).startswith("InvalidArgument:")


# ----------------------------------------------------------------------------- assemble
def test_cut_render_splats_matches_oracle(renderer, c1):
    h, oh, cam = c1
    cut = renderer.select_cut(h, cam, 3.0)
    g = renderer.cut_render_splats(h, cut)
    o = orc.cut_render_splats(oh, cut.node, cut.t, cut.alpha_prime)
    for f in ["mean", "scale", "rot_wxyz", "sh", "falloff", "parent_falloff", "t"]:
        assert np.array_equal(getattr(g, f).view(np.uint32), getattr(o, f).view(np.uint32)), f
    assert np.array_equal(g.siblings, o.siblings)


# ----------------------------------------------------------------------------- render_forward
@pytest.mark.parametrize("seed", range(4))
def test_render_forward_matches_oracle(renderer, seed):
    rng = Rng(200 + seed)
    sp = random_scene(rng, 150, True)
    cam = random_scene_camera(rng)
    out = renderer.render_forward(sp, cam, want_context=True)
    f = orc.render_forward(sp, cam)
    assert_images(out, f)
    check_projection(out, f)
    check_forward_context(out, f)


def test_render_forward_many_splats(renderer):
    rng = Rng(7)
    sp = random_scene(rng, 4000, True)
    cam = random_scene_camera(rng)
    out = renderer.render_forward(sp, cam, want_context=True)
    f = orc.render_forward(sp, cam)
    assert_images(out, f)
    check_forward_context(out, f)


def test_render_forward_empty(renderer):
    cam = hs.look_at_camera([0, 0, 0], [0, 0, 1], 40, 24, 60.0)
    out = renderer.render_forward(hs.RenderSplats.empty(0), cam)
    assert out.rendered_count == 0
    assert np.all(out.color == 0) and np.all(out.depth == 0) and np.all(out.transmittance == 1)


def test_render_forward_invalid_camera(renderer):
    cam = hs.look_at_camera([0, 0, 0], [0, 0, 1], 40, 24, 60.0)
    cam.fx = 0.0
    with pytest.raises(hs.Error) as e:
        renderer.render_forward(hs.RenderSplats.empty(0), cam)
    assert e.value.code == hs.Errc.InvalidArgument


# ----------------------------------------------------------------------------- render_hierarchy
def test_render_hierarchy_c1_bit_exact(renderer, c1):
    h, oh, cam = c1
    out, cut = renderer.render_hierarchy(h, cam, 3.0, want_context=True, return_cut=True)
    f = orc.render_hierarchy(oh, cam, 3.0)
    node, t, a = f.cut()
    assert np.array_equal(cut.node, node)
    assert_images(out, f)
    check_projection(out, f)
    check_forward_context(out, f)


def test_render_hierarchy_trajectory_c1(renderer, c1):
    h, oh, _ = c1
    cfg = scenes.CONFIGS["c1"]
    for cam in scenes.trajectory(cfg, 6, first=120):
        out = renderer.render_hierarchy(h, cam, cfg.tau)
        f = orc.render_hierarchy(oh, cam, cfg.tau, keep_ctx=False)
        assert_images(out, f)


def test_render_is_deterministic(renderer, c1):
    h, _, cam = c1
    a = renderer.render_hierarchy(h, cam, 3.0)
    b = renderer.render_hierarchy(h, cam, 3.0)
    assert np.array_equal(a.color.view(np.uint32), b.color.view(np.uint32))
    assert a.rendered_count == b.rendered_count


def test_fast_blend_within_tolerance(c1):
    h, oh, cam = c1
    r = hs.Renderer(0, exact=False)
    try:
        out = r.render_hierarchy(h, cam, 3.0)
    finally:
        pass
    f = orc.render_hierarchy(oh, cam, 3.0, keep_ctx=False)
    c, d, t, rc = f.images()
    assert np.abs(out.color - c).max() <= MAX_ABS
    assert np.abs(out.transmittance - t).max() <= MAX_ABS
    assert hs.psnr(out.color, c) >= MIN_PSNR
    r.close()


@pytest.fixture(scope="module")
def c1():
    cfg = scenes.CONFIGS["c1"]
    h = scenes.hierarchy(cfg)
    return h, orc.OracleHierarchy(h), scenes.camera(cfg, 130)
