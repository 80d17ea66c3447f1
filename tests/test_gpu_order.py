"""The per-tile depth order (bucket.cu) on adversarial tile loads, bit-exact
against the oracle: every size class and fallback of the in-tile sort.

  big tile, random depths        k_tile_split partitions (>= 4096 entries)
  big tile, one shared depth     a partition of > 4096 equal keys: chunks + merge
  regular tile, one shared depth MSD bucket > 64 -> LSD passes; ties by cut index
  small tile, one shared depth   the per-warp LSD fallback; ties by cut index
  many screen-covering splats    row difference marks, k_bucket_huge

The reference orders a tile's entries by (depth, cut index) (render.hpp:268-294,
stable_sort); equal depths are exactly where a non-stable device sort would
differ, so the shared-depth cases check the tie order too."""
import numpy as np
import pytest

import paper_2406_12080_b200 as hs
from oracle import oracle as orc
from tests.fixtures import Rng
from tests.test_gpu_parity import assert_images, check_forward_context

pytestmark = pytest.mark.gpu


def tile_cluster(rng, n, z, same_depth, px=(20.0, 20.0), focal=100.0, spread=4.0, sigma=0.004):
    """n small gray-ish splats projecting inside a few pixels around pixel px of a 64x48
    axis camera (z along +z): all land in one 16x16 tile."""
    cam = hs.look_at_camera([0, 0, 0], [0, 0, 1], 64, 48, focal)
    u = px[0] + rng.uniform(-spread, spread, n)
    v = px[1] + rng.uniform(-spread, spread, n)
    zz = np.full(n, z, np.float32) if same_depth else rng.uniform(z, 3 * z, n)
    x = (u - 32.0) * zz / focal
    y = (v - 24.0) * zz / focal
    mean = np.stack([x, -y, zz], 1).astype(np.float32)  # look_at: image y grows downwards
    scale = np.full((n, 3), sigma, np.float32) * zz[:, None]
    rot = np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1))
    sh = rng.uniform(-0.3, 0.3, (n, 48)).astype(np.float32)
    fall = rng.uniform(0.05, 0.2, n).astype(np.float32)
    return hs.RenderSplats.plain(mean, scale, rot, sh, fall), cam


def check(renderer, sp, cam):
    out = renderer.render_forward(sp, cam, want_context=True)
    f = orc.render_forward(sp, cam)
    assert_images(out, f)
    check_forward_context(out, f)
    return out


@pytest.mark.parametrize("n,same", [(12000, False), (9000, True), (3000, True), (400, True), (2500, False)])
def test_heavy_tile_orders_match_oracle(renderer, n, same):
    rng = Rng(1000 + n)
    sp, cam = tile_cluster(rng, n, 5.0, same)
    out = check(renderer, sp, cam)
    ts = out.context["tile_start"]
    assert np.diff(ts).max() >= n  # the cluster is one tile's list


def test_two_heavy_tiles_and_background(renderer):
    rng = Rng(77)
    a, cam = tile_cluster(rng, 6000, 4.0, False, px=(20.0, 20.0))
    b, _ = tile_cluster(rng, 5000, 6.0, True, px=(40.0, 28.0))
    c, _ = tile_cluster(rng, 3000, 3.0, False, px=(30.0, 24.0), spread=30.0)
    fields = ["mean", "scale", "rot_wxyz", "sh", "falloff", "parent_falloff", "t", "siblings"]
    sp = hs.RenderSplats(*[np.concatenate([getattr(s, k) for s in (a, b, c)]) for k in fields])
    check(renderer, sp, cam)


def test_screen_covering_splats(renderer):
    """Splats just in front of the image plane cover every tile (row marks, huge queue)."""
    rng = Rng(5)
    n = 300
    cam = hs.look_at_camera([0, 0, 0], [0, 0, 1], 320, 240, 200.0)
    zz = rng.uniform(0.02, 0.05, n)
    mean = np.stack([rng.uniform(-0.01, 0.01, n), rng.uniform(-0.01, 0.01, n), zz], 1).astype(np.float32)
    scale = np.full((n, 3), 0.05, np.float32)
    rot = np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1))
    sh = rng.uniform(-0.3, 0.3, (n, 48)).astype(np.float32)
    fall = rng.uniform(0.01, 0.03, n).astype(np.float32)
    sp = hs.RenderSplats.plain(mean, scale, rot, sh, fall)
    out = check(renderer, sp, cam)
    assert out.info["n_duplicates"] > 100 * n
