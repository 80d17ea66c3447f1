"""The CPU oracle pinned against the reference's own known-answer and
oracle-equivalence tests (ports of /root/reference/proj/tests/test_lod.cpp,
tests/test_render.cpp, tests/test_bench.cpp and tests/acceptance.cpp), with the
reference's tolerances.  CPU only."""
import math

import numpy as np
import pytest

import paper_2406_12080_b200 as hs
from oracle import oracle as orc
from tests.fixtures import (Rng, axis_camera, concat, descend, gray_splat, random_camera, random_hierarchy,
                            random_scene, random_scene_camera)

INF = float("inf")


def rel(a, b, tol):
    return abs(a - b) <= tol * abs(b)


# ----------------------------------------------------------------------------- test_lod.cpp
def test_granularity_pinhole_size():  # test_lod.cpp:55-72
    cam = hs.look_at_camera([0, 0, 0], [0, 0, 1], 640, 480, 500.0)
    assert rel(orc.granularity([-0.5, -0.1, 10.0], [0.5, 0.1, 10.0], cam), 50.0, 1e-5)
    assert rel(orc.granularity([-0.5, -0.1, 20.0], [0.5, 0.1, 20.0], cam), 25.0, 1e-5)
    assert rel(orc.granularity([-0.5, -0.5, 9.5], [0.5, 0.5, 10.5], cam), 500.0 / 9.5, 1e-5)


def test_granularity_nearest_corner_oracle():  # test_lod.cpp:74-100
    rng = Rng(60)
    for _ in range(200):
        cam = random_camera(rng, 4.0)
        a, b = rng.uniform(-5, 5, 3), rng.uniform(-5, 5, 3)
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        w = cam.world_to_camera.astype(np.float64)
        z_near = min(float(w[2, :3] @ np.array([(hi if k & 1 else lo)[0], (hi if k & 2 else lo)[1],
                                                 (hi if k & 4 else lo)[2]]) + w[2, 3]) for k in range(8))
        pos = cam.position()
        inside = bool(np.all(pos >= lo) and np.all(pos <= hi))
        got = orc.granularity(lo, hi, cam)
        if inside or z_near <= 0.01:
            assert got == INF
        else:
            assert rel(got, cam.fx * float(np.max(hi - lo)) / z_near, 1e-4)


def test_granularity_inside_or_behind():  # test_lod.cpp:102-113
    cam = hs.look_at_camera([0, 0, 0], [0, 0, 1], 640, 480, 500.0)
    assert orc.granularity([-1, -1, -1], [1, 1, 1], cam) == INF
    assert orc.granularity([-1, -1, -5], [1, 1, -4], cam) == INF


def test_granularity_monotone_parent_child():  # test_lod.cpp:115-128
    rng = Rng(61)
    for _ in range(8):
        h = random_hierarchy(rng, 64)
        for _ in range(12):
            cam = random_camera(rng, 5.0)
            for i in range(1, h.n):
                p = h.parent[i]
                assert orc.granularity(h.bmin[p], h.bmax[p], cam) >= orc.granularity(h.bmin[i], h.bmax[i], cam)


def test_interp_weight_values():  # test_lod.cpp:130-141
    assert orc.interp_weight(4.0, 8.0, 4.0) == 1.0
    assert orc.interp_weight(4.0, 8.0, 8.0) == 0.0
    assert orc.interp_weight(4.0, 8.0, 6.0) == 0.5
    assert orc.interp_weight(4.0, 8.0, 2.0) == 1.0
    assert orc.interp_weight(4.0, 8.0, 99.0) == 0.0
    assert orc.interp_weight(5.0, 5.0, 3.0) == 1.0
    assert orc.interp_weight(3.0, INF, 7.0) == 1.0


def test_transition_alpha_composes():  # test_lod.cpp:143-158
    assert abs(orc.transition_alpha(0.75, 2) - 0.5) <= 1e-6
    assert abs(orc.transition_alpha(0.36, 1) - 0.36) <= 1e-6
    rng = Rng(62)
    for _ in range(100):
        a = float(rng.uniform(0.0, 0.99))
        k = 1 + rng.randint(6)
        ap = np.float32(orc.transition_alpha(a, k))
        assert abs(float(1.0 - np.float32(np.float32(1.0 - ap) ** np.float32(k))) - a) <= 1e-5
    assert orc.transition_alpha(5.0, 2) == orc.transition_alpha(0.99, 2)
    with pytest.raises(orc.OracleError):
        orc.transition_alpha(0.5, 0)


def test_cut_matches_recursive_descent():  # test_lod.cpp:160-174, acceptance.cpp:183-241
    rng = Rng(63)
    for _ in range(60):
        h = random_hierarchy(rng, 1 + rng.randint(128))
        cam = random_camera(rng, 5.0)
        tau = float(rng.uniform(0.5, 400.0))
        node, _, _ = orc.select_cut(orc.OracleHierarchy(h), cam, tau)
        assert list(node) == descend(h, cam, tau, orc.granularity)


def test_cut_partitions_leaves():  # test_lod.cpp:176-199
    rng = Rng(64)
    h = random_hierarchy(rng, 200)
    oh = orc.OracleHierarchy(h)
    for _ in range(10):
        cam = random_camera(rng, 5.0)
        node, _, _ = orc.select_cut(oh, cam, float(rng.uniform(1.0, 300.0)))
        covered = np.zeros(h.n, np.int32)
        for e in node:
            stack = [int(e)]
            while stack:
                i = stack.pop()
                if h.child_count[i] == 0:
                    covered[i] += 1
                stack.extend(range(int(h.first_child[i]), int(h.first_child[i] + h.child_count[i])))
        assert np.all(covered[h.child_count == 0] == 1)


def test_zero_threshold_selects_leaves():  # test_lod.cpp:201-212
    rng = Rng(65)
    h = random_hierarchy(rng, 75)
    node, t, _ = orc.select_cut(orc.OracleHierarchy(h), random_camera(rng, 5.0), 0.0)
    assert np.array_equal(node, np.flatnonzero(h.child_count == 0))
    assert np.all(t == 1.0)


def test_huge_threshold_selects_root():  # test_lod.cpp:214-222
    rng = Rng(66)
    h = random_hierarchy(rng, 75)
    cam = hs.look_at_camera([0, 0, -400], [0, 0, 0], 64, 64, 100.0)
    node, t, _ = orc.select_cut(orc.OracleHierarchy(h), cam, 1e9)
    assert list(node) == [0] and t[0] == 1.0


def test_cut_entries_carry_split_opacity():  # test_lod.cpp:224-241
    rng = Rng(67)
    h = random_hierarchy(rng, 90)
    node, t, a = orc.select_cut(orc.OracleHierarchy(h), random_camera(rng, 5.0), 24.0)
    assert np.all((t >= 0) & (t <= 1))
    for n, tv, av in zip(node, t, a):
        if n == 0:
            assert tv == 1.0
            continue
        p = h.parent[n]
        assert abs(av - orc.transition_alpha(float(h.falloff[p]), int(h.child_count[p]))) <= 1e-6


def test_assembled_splats_expose_blend_inputs():  # test_lod.cpp:267-292
    rng = Rng(69)
    h = random_hierarchy(rng, 120)
    oh = orc.OracleHierarchy(h)
    node, t, a = orc.select_cut(oh, random_camera(rng, 5.0), 16.0)
    sp = orc.cut_render_splats(oh, node, t, a)
    assert len(sp) == len(node)
    for i, n in enumerate(node):
        assert sp.t[i] == t[i] or (n == 0 or t[i] >= 1.0)
        if n == 0 or t[i] >= 1.0:
            assert np.array_equal(sp.mean[i], h.mean[n]) and sp.falloff[i] == h.falloff[n] and sp.siblings[i] == 1
        else:
            p = h.parent[n]
            assert sp.siblings[i] == h.child_count[p]
            assert sp.parent_falloff[i] == h.falloff[p] and sp.falloff[i] == h.falloff[n]
            np.testing.assert_allclose(sp.mean[i], t[i] * h.mean[n] + (1 - t[i]) * h.mean[p], rtol=1e-5, atol=1e-5)


# ----------------------------------------------------------------------------- test_render.cpp
def test_projection_on_axis_closed_form():  # test_render.cpp:71-87
    f, z, sigma = 80.0, 5.0, 0.3
    o, cov, dets = orc.project(gray_splat([0, 0, z], sigma, 0.7), axis_camera(64, 64, f))
    assert o[0] == 0
    s2 = (f * sigma / z) ** 2
    assert rel(cov[0], s2 + 0.3, 1e-5) and rel(cov[3], s2 + 0.3, 1e-5) and abs(cov[1]) <= 1e-4
    assert rel(dets[0], s2 * s2, 1e-4)
    assert rel(o[7], s2 / (s2 + 0.3), 1e-5)
    assert abs(o[2] - 32.0) <= 1e-4 and abs(o[3] - 32.0) <= 1e-4
    assert rel(o[11], 1.0 / z, 1e-6)
    assert o[12:13].view(np.int32)[0] == int(math.ceil(3.0 * math.sqrt(np.float32(s2 + 0.3))))


def test_projection_small_angle():  # test_render.cpp:89-101
    f, z, sigma = 300.0, 20.0, 0.02
    o, cov, _ = orc.project(gray_splat([0.4, -0.3, z], sigma, 0.7), axis_camera(128, 128, f))
    s2 = (f * sigma / z) ** 2
    assert rel(cov[0] - 0.3, s2, 1e-2) and rel(cov[3] - 0.3, s2, 1e-2) and abs(cov[1]) < 1e-2 * s2


def test_band0_radiance_clamped():  # test_render.cpp:103-122
    sp = gray_splat([0.5, -0.2, 6.0], 0.2, 1.0)
    sp.sh[0, 0], sp.sh[0, 1], sp.sh[0, 2] = 1.1, -0.4, -2.5
    c0 = 0.28209479177387814
    expect = [0.5 + c0 * 1.1, 0.5 + c0 * -0.4, 0.0]
    for pos in ([0, 0, 0], [3, 1, 0], [-2, -4, 1]):
        o, _, _ = orc.project(sp, hs.look_at_camera(pos, [0.5, -0.2, 6.0], 64, 64, 90.0))
        assert o[0] == 0
        np.testing.assert_allclose(o[8:11], expect, atol=1e-5)


def test_dilation_alpha_scale():  # test_render.cpp:124-133
    cam = axis_camera(64, 64, 100.0)
    assert orc.project(gray_splat([0, 0, 2], 4.0, 0.5), cam)[0][7] > 0.999
    assert orc.project(gray_splat([0, 0, 40], 0.01, 0.5), cam)[0][7] < 0.1


def test_projection_culls():  # test_render.cpp:135-144
    cam = axis_camera(64, 64, 100.0)
    assert orc.project(gray_splat([0, 0, -3], 0.3, 0.7), cam)[0][0] == 1
    assert orc.project(gray_splat([0, 0, 0.005], 0.3, 0.7), cam)[0][0] == 1
    assert orc.project(gray_splat([50, 0, 5], 0.1, 0.7), cam)[0][0] == 1
    bad = gray_splat([0, 0, 5], 0.3, 0.7)
    bad.rot_wxyz[:] = 0
    assert orc.project(bad, cam)[0][0] == 1


def test_single_splat_pixel_oracle():  # test_render.cpp:146-183
    f, z, sigma, falloff = 80.0, 5.0, 0.3, 0.6
    fr = orc.render_forward(gray_splat([0, 0, z], sigma, falloff), axis_camera(64, 64, f))
    color, depth, trans, rc = fr.images()
    s2 = (f * sigma / z) ** 2
    var = s2 + 0.3
    ascale = s2 / var
    radius = int(math.ceil(3.0 * math.sqrt(var)))
    t0, t1 = (32 - radius) // 16, (32 + radius) // 16 + 1
    contributing = 0
    for y in range(64):
        for x in range(64):
            alpha = 0.0
            if t0 <= x // 16 < t1 and t0 <= y // 16 < t1:
                dx, dy = x + 0.5 - 32.0, y + 0.5 - 32.0
                a = min(0.99, falloff * ascale * math.exp(-0.5 * (dx * dx + dy * dy) / var))
                assert abs(a - 1 / 255) > 5e-6
                if a >= 1 / 255:
                    alpha = a
                    contributing += 1
            assert abs(color[0, y, x] - 0.5 * alpha) <= 2e-6 and abs(color[1, y, x] - 0.5 * alpha) <= 2e-6
            assert abs(depth[y, x] - alpha / z) <= 2e-6
            assert abs(trans[y, x] - (1 - alpha)) <= 2e-6
    assert contributing > 200 and rc == 1


def test_depth_is_weight_times_inverse_depth():  # test_render.cpp:185-196
    z = 7.0
    color, depth, trans, _ = orc.render_forward(gray_splat([0, 0, z], 0.4, 0.8), axis_camera(48, 48, 70.0)).images()
    np.testing.assert_allclose(depth, (1.0 - trans) / z, atol=1e-6)


def test_input_order_invariance():  # test_render.cpp:198-218
    rng = Rng(70)
    cam = axis_camera(64, 48, 90.0)
    parts = []
    for _ in range(20):
        m = rng.uniform(-1, 1, 3)
        m[2] = rng.uniform(4.0, 9.0)
        parts.append(gray_splat(m, float(rng.uniform(0.1, 0.4)), float(rng.uniform(0.3, 0.9))))
    a = concat(parts)
    b = concat(parts[::-1])
    ia, ib = orc.render_forward(a, cam).images(), orc.render_forward(b, cam).images()
    for k in range(3):
        assert np.array_equal(ia[k].view(np.uint32), ib[k].view(np.uint32))
    assert ia[3] == ib[3]


def test_tiled_equals_naive_bitwise():  # test_render.cpp:220-232, acceptance.cpp:529-561
    rng = Rng(71)
    for _ in range(4):
        sp = random_scene(rng, 150, True)
        cam = random_scene_camera(rng)
        t = orc.render_forward(sp, cam).images()
        n = orc.render_reference(sp, cam).images()
        for k in range(3):
            assert np.array_equal(t[k].view(np.uint32), n[k].view(np.uint32))
        assert t[3] == n[3]


def test_empty_scene():  # test_render.cpp:234-241
    c, d, t, rc = orc.render_forward(hs.RenderSplats.empty(0), axis_camera(40, 24, 60.0)).images()
    assert rc == 0 and np.all(c == 0) and np.all(d == 0) and np.all(t == 1)


def test_falloff_saturates_and_negative_is_invisible():  # test_render.cpp:243-261
    cam = axis_camera(64, 64, 80.0)
    for big in (4.0, 1e8):
        c, d, t, _ = orc.render_forward(gray_splat([0, 0, 5], 0.3, big), cam).images()
        assert np.all(np.isfinite(c)) and np.all(np.isfinite(d)) and np.all(np.isfinite(t))
        assert abs(t[32, 32] - (1 - 0.99)) <= 1e-6
    c, d, t, rc = orc.render_forward(gray_splat([0, 0, 5], 0.3, -0.5), cam).images()
    assert rc == 0 and np.all(t == 1)


def test_coverage_never_exceeds_one():  # test_render.cpp:263-283
    rng = Rng(72)
    sp = random_scene(rng, 120, True)
    white = 0.5 / 0.28209479177387814
    sp.sh[:] = 0
    sp.sh[:, :3] = white
    c, d, t, _ = orc.render_forward(sp, random_scene_camera(rng)).images()
    assert np.all((t >= 0) & (t <= 1))
    np.testing.assert_allclose(c[0], 1.0 - t, atol=1e-5)
    assert np.all(c[0] <= 1 + 1e-6)


def test_transition_blends_two_laws():  # test_render.cpp:285-309
    cam = axis_camera(48, 48, 70.0)
    s = gray_splat([0, 0, 6], 0.5, 0.8)
    s.t[0], s.parent_falloff[0], s.siblings[0] = 0.4, 0.6, 3
    c, d, t, _ = orc.render_forward(s, cam).images()
    o, _, _ = orc.project(s, cam)
    for y in range(48):
        for x in range(48):
            dx, dy = x + 0.5 - o[2], y + 0.5 - o[3]
            g = math.exp(-0.5 * (o[4] * dx * dx + o[6] * dy * dy) - o[5] * dx * dy)
            self_ = min(0.99, 0.8 * o[7] * g)
            par = min(0.99, 0.6 * o[7] * g)
            self_ = 0.0 if self_ < 1 / 255 else self_
            split = 1 - (1 - par) ** (1 / 3) if par >= 1 / 255 else 0.0
            assert abs((1 - t[y, x]) - (0.4 * self_ + 0.6 * split)) <= 1e-5


def test_children_at_transition_start_reproduce_parent():  # test_render.cpp:311-355, acceptance.cpp:133-181
    rng = Rng(73)
    from tests.fixtures import random_gaussians
    for k in (2, 3, 5):
        mean, scale, rot, fall, sh = random_gaussians(rng, k, 1.0, 0.2, 0.6, 0.3, 0.95)
        leaves = hs.build_bvh(mean, scale, rot, fall, sh)  # gives a merged parent for the root
        root = 0
        # one parent, k children at t = 0 (hand-built like the reference)
        h = hs.Hierarchy.empty(k + 1)
        for name in ("mean", "scale", "rot_wxyz", "falloff", "sh"):
            getattr(h, name)[0] = getattr(leaves, name)[root]
            getattr(h, name)[1:] = {"mean": mean, "scale": scale, "rot_wxyz": rot, "falloff": fall, "sh": sh}[name]
        h.parent[:] = 0
        h.parent[0] = hs.NO_NODE
        h.first_child[:] = hs.NO_NODE
        h.first_child[0] = 1
        h.child_count[0] = k
        h.bmin[:] = -100
        h.bmax[:] = 100
        oh = orc.OracleHierarchy(h)
        node = np.arange(1, k + 1, dtype=np.uint32)
        children = orc.cut_render_splats(oh, node, np.zeros(k, np.float32))
        parent = hs.RenderSplats.plain(h.mean[:1], h.scale[:1], h.rot_wxyz[:1], h.sh[:1], h.falloff[:1])
        cam = hs.look_at_camera([1.5, 1.0, -7.0], h.mean[0], 96, 96, 140.0)
        a = orc.render_forward(children, cam).images()
        b = orc.render_forward(parent, cam).images()
        np.testing.assert_allclose(a[0], b[0], atol=1e-5)
        np.testing.assert_allclose(a[2], b[2], atol=1e-5)


def test_hierarchy_pipeline_timings():  # test_render.cpp:641-659
    rng = Rng(78)
    from tests.fixtures import random_gaussians
    h = hs.build_bvh(*random_gaussians(rng, 80, 3.0, 0.1, 0.5, 0.3, 1.0))
    cam = hs.look_at_camera([9, 5, -9], [0, 0, 0], 96, 80, 110.0)
    fr = orc.render_hierarchy(orc.OracleHierarchy(h), cam, 8.0)
    c, d, t, rc = fr.images()
    assert np.all(np.isfinite(c)) and rc > 0 and rc <= fr.sizes()["ncut"]
    assert all(v >= 0 for v in fr.times().values())


# ----------------------------------------------------------------------------- test_bench.cpp
def test_psnr_closed_forms():  # test_bench.cpp:40-63
    rng = Rng(21)
    img = rng.uniform(0, 1, (3, 24, 32))
    assert hs.psnr(img, img) == 99.0
    amp = 0.01 * math.sqrt(3.0)
    ref = rng.uniform(0.2, 0.8, (3, 128, 128))
    noisy = (ref + rng.uniform(-amp, amp, ref.shape)).astype(np.float32)
    assert abs(hs.psnr(noisy, ref) - 40.0) <= 0.1
    with pytest.raises(hs.Error) as e:
        hs.psnr(np.zeros((3, 4, 4), np.float32), np.zeros((3, 5, 4), np.float32))
    assert e.value.code == hs.Errc.DimensionMismatch


def test_bench_path_accounting():  # test_bench.cpp:87-139
    rng = Rng(22)
    from tests.fixtures import random_gaussians
    h = hs.build_bvh(*random_gaussians(rng, 128, 4.0, 0.05, 0.2, 0.3, 0.9))
    oh = orc.OracleHierarchy(h)
    cam_at = lambda z: hs.look_at_camera([0, 0, z], [0, 0, 0], 64, 48, 60.0)  # noqa: E731
    st = orc.bench_path(oh, [cam_at(-30.0)] * 6, 2.0)
    assert st[0, 0] > 0 and st[0, 2] == st[0, 0]
    assert np.all(st[1:, 0] == st[0, 0]) and np.all(st[1:, 2] == 0)
    assert np.all(st[1::2, 3] == 0) and np.all(st[1::2, 4] == 0)
    st0 = orc.bench_path(oh, [cam_at(-30.0)] * 2, 0.0)
    assert np.all(st0[:, 0] == 128) and np.all(st0[:, 1] == 100.0)
    st2 = orc.bench_path(oh, [cam_at(-40.0), cam_at(-40.0), cam_at(-2.5), cam_at(-2.5)], 4.0)
    assert st2[2, 0] > st2[0, 0] and st2[2, 2] > 0 and st2[3, 2] == 0
