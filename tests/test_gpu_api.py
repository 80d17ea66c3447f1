"""The reference's per-object API on the device (C ABI -> lodapi.cu kernels)
against the oracle, bit for bit: granularity / interp_weight /
transition_alpha (lod.hpp:18-45), interpolated_gaussian (lod.hpp:97-110),
assemble_cut_splats over caller attributes (lod.hpp:116-146), project
(render.hpp:104-176), render_reference (render.hpp:360-408) and
ForwardContext::order (render.hpp:93)."""
import numpy as np
import pytest

import paper_2406_12080_b200 as hs
from oracle import oracle as orc
from tests.fixtures import Rng, axis_camera, gray_splat, random_camera, random_hierarchy, random_scene, \
    random_scene_camera

pytestmark = pytest.mark.gpu


def u32(a):
    return np.asarray(a, np.float32).view(np.uint32)


def test_granularity_matches_oracle(renderer):
    rng = Rng(60)
    for _ in range(20):
        cam = random_camera(rng, 4.0)
        a = rng.uniform(-5.0, 5.0, (64, 3))
        b = rng.uniform(-5.0, 5.0, (64, 3))
        bmin, bmax = np.minimum(a, b), np.maximum(a, b)
        got = renderer.granularity(bmin, bmax, cam)
        want = np.array([orc.granularity(bmin[i], bmax[i], cam) for i in range(64)], np.float32)
        assert np.array_equal(u32(got), u32(want))
    # inside / behind -> inf (test_lod.cpp:102-113)
    cam = axis_camera(640, 480, 500.0)
    assert hs.granularity([-1, -1, -1], [1, 1, 1], cam) == np.inf
    assert hs.granularity([-1, -1, -5], [1, 1, -4], cam) == np.inf


def test_interp_weight_and_transition_alpha_match_oracle(renderer):
    rng = Rng(61)
    en = rng.uniform(0.0, 50.0, 500)
    ep = en + rng.uniform(0.0, 50.0, 500)
    ep[::7] = np.inf
    ep[::11] = en[::11]
    tau = 17.0
    got = renderer.interp_weight(en, ep, tau)
    want = np.array([orc.interp_weight(float(x), float(y), tau) for x, y in zip(en, ep)], np.float32)
    assert np.array_equal(u32(got), u32(want))
    a = np.concatenate([rng.uniform(-0.5, 1.5, 400), [0.0, 0.99, 5.0]]).astype(np.float32)
    k = np.array([1 + rng.randint(17) for _ in range(len(a))], np.int32)
    got = renderer.transition_alpha(a, k)
    want = np.array([orc.transition_alpha(float(x), int(kk)) for x, kk in zip(a, k)], np.float32)
    assert np.array_equal(u32(got), u32(want))
    assert hs.transition_alpha(0.75, 2) == pytest.approx(0.5, abs=1e-6)
    with pytest.raises(hs.Error) as e:
        hs.transition_alpha(0.5, 0)
    assert e.value.code == hs.Errc.InvalidArgument


def _gauss(rng, n):
    m, s, r, f, sh = (np.ascontiguousarray(x) for x in
                      __import__("tests.fixtures", fromlist=["random_gaussians"]).random_gaussians(rng, n))
    return {"mean": m, "scale": s, "rot_wxyz": r, "falloff": f, "sh": sh}


def test_interpolated_gaussian_endpoints(renderer):
    """test_lod.cpp:243-265: t = 1 is the child; t = 0 the parent's shape with the split alpha."""
    rng = Rng(68)
    c, p = _gauss(rng, 50), _gauss(rng, 50)
    at1 = renderer.interpolated_gaussian(c, p, 1.0, 2)
    for k in ("mean", "scale", "falloff", "sh"):
        assert np.array_equal(at1[k], c[k]), k
    dots = np.abs(np.sum(at1["rot_wxyz"] * c["rot_wxyz"], axis=1))
    assert np.all(dots > 1.0 - 1e-6)
    at0 = renderer.interpolated_gaussian(c, p, 0.0, 3)
    for k in ("mean", "scale", "sh"):
        assert np.array_equal(at0[k], p[k]), k
    split = renderer.transition_alpha(np.minimum(p["falloff"], 0.99), 3)
    assert np.array_equal(u32(at0["falloff"]), u32(split))
    mid = renderer.interpolated_gaussian(c, p, 0.5, 2)
    assert np.allclose(mid["mean"], 0.5 * (c["mean"] + p["mean"]), atol=1e-6)
    assert np.allclose(np.linalg.norm(mid["rot_wxyz"], axis=1), 1.0, atol=1e-6)


def test_assemble_cut_splats_over_caller_attributes(renderer):
    """Over the hierarchy's own attributes it is cut_render_splats (lod.hpp:148-153); over
    other attribute arrays it blends those; a mismatched array is DimensionMismatch."""
    rng = Rng(69)
    h = random_hierarchy(rng, 300)
    cam = random_camera(rng, 5.0)
    cut = renderer.select_cut(h, cam, 16.0)
    ref = renderer.cut_render_splats(h, cut)
    attrs = {"mean": h.mean, "scale": h.scale, "rot_wxyz": h.rot_wxyz, "falloff": h.falloff, "sh": h.sh}
    got = renderer.assemble_cut_splats(h, attrs, cut)
    for k in ("mean", "scale", "rot_wxyz", "sh", "falloff", "parent_falloff", "t", "siblings"):
        assert np.array_equal(np.asarray(getattr(got, k)).view(np.uint32), np.asarray(getattr(ref, k)).view(np.uint32)), k
    # trainable copies (refine.hpp:316-317): shifted means blend the same way
    moved = dict(attrs, mean=(h.mean + np.float32(0.25)).astype(np.float32))
    got2 = renderer.assemble_cut_splats(h, moved, cut)
    plain = cut.t >= 1.0
    assert np.array_equal(got2.mean[plain], moved["mean"][cut.node[plain]])
    with pytest.raises(hs.Error) as e:
        renderer.assemble_cut_splats(h, {k: v[:-1] for k, v in attrs.items()}, cut)
    assert e.value.code == hs.Errc.DimensionMismatch


def test_project_matches_oracle(renderer):
    rng = Rng(72)
    for _ in range(3):
        sp = random_scene(rng, 40, True)
        cam = random_scene_camera(rng)
        got = renderer.project(sp, cam)
        for i in range(len(sp)):
            one = hs.RenderSplats(*[getattr(sp, f)[i:i + 1] for f in ("mean", "scale", "rot_wxyz", "sh", "falloff",
                                                                       "parent_falloff", "t", "siblings")])
            p16, cov, dets = orc.project(one, cam)
            g = got[i]
            assert bool(g["culled"]) == bool(p16[0] != 0)
            if g["culled"]:
                continue
            assert u32(g["cam_point"][2]) == u32(p16[1])
            assert np.array_equal(u32(g["mean2d"]), u32(p16[2:4]))
            assert np.array_equal(u32(g["conic"]), u32(p16[4:7]))
            assert u32(g["alpha_scale"]) == u32(p16[7])
            assert np.array_equal(u32(g["color"]), u32(p16[8:11]))
            assert u32(g["inv_depth"]) == u32(p16[11])
            assert int(g["radius"]) == int(p16[12:13].view(np.int32)[0])
            assert np.array_equal(u32(g["cov2d"]), u32(cov))
            assert u32(g["det_pre"]) == u32(dets[0]) and u32(g["det_post"]) == u32(dets[1])
    # culling cases (test_render.cpp:135-144)
    cam = axis_camera(64, 64, 100.0)
    for mean in ([0, 0, -3], [0, 0, 0.005], [50, 0, 5]):
        assert renderer.project(gray_splat(mean, 0.3, 0.7), cam)[0]["culled"]


def test_render_reference_equals_tiled_and_oracle(renderer):
    """test_render.cpp:220-232 on the device: the naive renderer equals the tiled one bit
    for bit; both equal the oracle's render_reference."""
    rng = Rng(71)
    for _ in range(4):
        sp = random_scene(rng, 150, True)
        cam = random_scene_camera(rng)
        tiled = renderer.render_forward(sp, cam)
        naive = renderer.render_reference(sp, cam)
        f = orc.render_reference(sp, cam)
        c, d, T, rc = f.images()
        for got in (tiled, naive):
            assert np.array_equal(got.color.view(np.uint32), c.view(np.uint32))
            assert np.array_equal(got.depth.view(np.uint32), d.view(np.uint32))
            assert np.array_equal(got.transmittance.view(np.uint32), T.view(np.uint32))
            assert got.rendered_count == rc


def test_forward_context_order_is_the_stable_depth_order(renderer):
    rng = Rng(73)
    sp = random_scene(rng, 200, True)
    cam = random_scene_camera(rng)
    out = renderer.render_forward(sp, cam, want_context=True)
    f = orc.render_forward(sp, cam, keep_ctx=True)
    assert np.array_equal(out.context["order"], f.context()["order"])
