"""The reference's acceptance criteria on the hot path (tests/acceptance.cpp),
run through the GPU path: #3 cuts equal the recursive-descent reference and
partition the leaves (acceptance.cpp:183-241), #5 coarse cuts render at most
half the leaves (:279-289), #11 cut time grows at most linearly with the node
count (:626-684), and the tau = 0 hierarchy render equals the leaf render
(test_bench.cpp:175-198)."""
import time

import numpy as np
import pytest

import paper_2406_12080_b200 as hs
from oracle import oracle as orc
from paper_2406_12080_b200 import scenes
from tests.fixtures import Rng, descend, random_camera, random_hierarchy

pytestmark = pytest.mark.gpu


def _leaves_under(h, nodes):
    out = []
    for nd in nodes:
        stack = [int(nd)]
        while stack:
            i = stack.pop()
            if h.child_count[i] == 0:
                out.append(i)
            else:
                stack.extend(range(int(h.first_child[i]), int(h.first_child[i] + h.child_count[i])))
    return sorted(out)


def test_acceptance3_cuts_equal_recursive_descent(renderer):
    """100 trees of <= 512 leaves x 10 cameras x tau in {1, 3, 6, 15} = 4000 cuts."""
    rng = Rng(2031)
    checked = 0
    for _ in range(100):
        h = random_hierarchy(rng, 1 + rng.randint(512))
        dh = renderer.upload(h)
        leaves = list(np.flatnonzero(h.child_count == 0))
        for _ in range(10):
            cam = random_camera(rng, 5.0)
            for tau in (1.0, 3.0, 6.0, 15.0):
                cut = renderer.select_cut(dh, cam, tau).node
                assert list(cut) == descend(h, cam, tau, orc.granularity)
                assert _leaves_under(h, cut) == leaves  # the cut partitions the leaves
                checked += 1
    assert checked == 4000


def test_acceptance5_coarse_cut_renders_at_most_half(renderer):
    cfg = scenes.Config("toy", 5040, 320, 240, 200.0, 15.0, altitude=12.0, standoff=10.0, lookahead=40.0)
    h = hs.synth_city(cfg.leaves, seed=5)
    rep = hs.bench_path(h, scenes.trajectory(cfg, 6, first=0), 15.0, renderer=renderer)
    assert rep.mean_rendered_pct <= 50.0


def test_acceptance11_cut_time_at_most_linear(renderer):
    """log-log slope of cut time over 1e4..1e6 nodes <= 1.3 (acceptance.cpp:626-684)."""
    sizes, times = [], []
    for leaves in (5_000, 50_000, 500_000):
        h = hs.synth_city(leaves, seed=7)
        dh = renderer.upload(h, validate=False)
        cam = scenes.camera(scenes.Config("s", leaves, 640, 480, 300.0, 3.0), 10)
        renderer.select_cut_device(dh, cam, 3.0)
        t0 = time.perf_counter()
        for _ in range(20):
            renderer.select_cut_device(dh, cam, 3.0)
        times.append((time.perf_counter() - t0) / 20)
        sizes.append(dh.n)
    slope = np.polyfit(np.log(sizes), np.log(times), 1)[0]
    assert slope <= 1.3, (sizes, times)


def test_tau_zero_hierarchy_render_equals_leaf_render(renderer):  # test_bench.cpp:175-198
    h = hs.synth_city(3000, seed=12)
    cfg = scenes.Config("t0", 3000, 160, 120, 90.0, 0.0, altitude=10.0, standoff=8.0, lookahead=30.0)
    cam = scenes.camera(cfg, 50)
    out = renderer.render_hierarchy(h, cam, 0.0)
    leaf = np.flatnonzero(h.child_count == 0)
    sp = hs.RenderSplats.plain(h.mean[leaf], h.scale[leaf], h.rot_wxyz[leaf], h.sh[leaf], h.falloff[leaf])
    ref = renderer.render_forward(sp, cam)
    assert hs.psnr(out.color, ref.color) >= 60.0
