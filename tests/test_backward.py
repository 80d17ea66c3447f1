"""render_backward (render.hpp:427-702).  CPU: the oracle's
float restatement against the reference's own gradient tests
(tests/test_render.cpp:465-643: central finite differences, the band-0 closed
form, the exposure outer products, the saturated-alpha freeze).  GPU:
hs_render_backward against the oracle within a tolerance (the two sum in
different orders), and run-to-run determinism."""
import copy

import numpy as np
import pytest

import paper_2406_12080_b200 as hs
from oracle import oracle as orc
from tests.fixtures import Rng, axis_camera, gray_splat, random_scene, random_scene_camera

GRAD_KEYS = ("mean", "scale", "rotation", "falloff", "parent_falloff", "t", "sh", "mean2d")
EXPO = np.array([[1.2, 0.05, 0.0, 0.02], [0.0, 0.9, -0.04, -0.03], [0.03, 0.0, 1.05, 0.01]], np.float32)


def grad_fixture():
    """make_grad_fixture (test_render.cpp:398-433): 5 splats, 2 in transition."""
    rng = Rng(75)
    n = 5
    mean = np.stack([rng.uniform(-1.2, 1.2, n), rng.uniform(-1.2, 1.2, n), rng.uniform(4.5, 8.0, n)], 1)
    scale = rng.uniform(0.15, 0.5, (n, 3))
    q = rng.uniform(-1.0, 1.0, (n, 4))
    q = (q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32)
    sh = np.zeros((n, 48), np.float32)
    sh[:, :3] = rng.uniform(0.9, 1.5, (n, 3))
    sh[:, 3:] = rng.uniform(-0.06, 0.06, (n, 45))
    sp = hs.RenderSplats.plain(mean.astype(np.float32), scale, q, sh, rng.uniform(0.3, 0.8, n))
    for i, (t, k) in ((3, (0.35, 2)), (4, (0.7, 3))):
        sp.t[i] = t
        sp.parent_falloff[i] = rng.uniform(0.3, 0.8)
        sp.siblings[i] = k
    cam = axis_camera(32, 32, 40.0)
    lw = rng.uniform(-1.0, 1.0, (3, 32, 32))
    dw = rng.uniform(-1.0, 1.0, (32, 32))
    return sp, cam, lw, dw


def loss(sp, cam, lw, dw):
    """fixture_loss (test_render.cpp:437-449): weighted exposed colour + inverse depth, in double."""
    f = orc.render_forward(sp, cam, keep_ctx=False)
    c, d, _, _ = f.images()
    cd = c.astype(np.float64).reshape(3, -1)
    exposed = EXPO[:, :3].astype(np.float64) @ cd + EXPO[:, 3:4].astype(np.float64)
    return float((lw.astype(np.float64).reshape(3, -1) * exposed).sum() + (dw.astype(np.float64) * d).sum())


def test_autograd_reference_matches_finite_differences():  # test_render.cpp:465-554, in float64
    """The float64 autograd restatement (tests/torch_ref.py) passes the reference's own
    finite-difference criterion: 299 coordinates, >= 95% within 2% (h = 1e-4 max(|v|, 0.1))."""
    import torch
    from tests import torch_ref
    sp, cam, lw, dw = grad_fixture()
    g = torch_ref.gradients(sp, cam, lw, dw, EXPO)
    base = {"mean": sp.mean, "scale": sp.scale, "rot": sp.rot_wxyz, "sh": sp.sh, "falloff": sp.falloff,
            "parent_falloff": sp.parent_falloff, "t": sp.t}
    key_of = {"mean": "mean", "scale": "scale", "rot": "rotation", "sh": "sh", "falloff": "falloff",
              "parent_falloff": "parent_falloff", "t": "t"}

    def loss(p):
        with torch.no_grad():
            c, d = torch_ref.render(p, cam, EXPO)
            return float((torch.tensor(lw, dtype=torch.float64) * c).sum() +
                         (torch.tensor(dw, dtype=torch.float64) * d).sum())

    def params():
        p = {k: torch.tensor(np.asarray(v, np.float64)) for k, v in base.items()}
        p["inv_k"] = torch.tensor(1.0 / np.maximum(1, sp.siblings).astype(np.float64))
        return p

    passed = total = 0
    for i in range(5):
        probes = [(k, j) for k, m in (("mean", 3), ("scale", 3), ("rot", 4), ("falloff", 1), ("sh", 48))
                  for j in range(m)]
        if sp.t[i] < 1.0:
            probes += [("parent_falloff", 0), ("t", 0)]
        for k, j in probes:
            v = float(base[k][i, j] if base[k].ndim == 2 else base[k][i])
            h = 1e-4 * max(abs(v), 0.1)
            vals = []
            for sgn in (1.0, -1.0):
                p = params()
                if p[k].ndim == 2:
                    p[k][i, j] += sgn * h
                else:
                    p[k][i] += sgn * h
                vals.append(loss(p))
            fd = (vals[0] - vals[1]) / (2 * h)
            gk = g[key_of[k]]
            an = float(gk[i, j] if gk.ndim == 2 else gk[i])
            total += 1
            denom = max(abs(an), abs(fd), 1e-7)
            if (abs(an) < 1e-12 and abs(fd) < 1e-12) or abs(an - fd) / denom <= 0.02:
                passed += 1
    assert total == 299  # 59 per splat + 2 per transition splat (test_render.cpp:544)
    assert passed >= 0.95 * total, f"{passed} of {total} within 2%"


@pytest.mark.parametrize("case", ["fixture", "scene77", "scene81"])
def test_oracle_gradients_match_autograd(case):
    """The oracle's float render_backward against float64 autograd of the same renderer."""
    from tests import torch_ref
    if case == "fixture":
        sp, cam, lw, dw = grad_fixture()
        ex = EXPO
    else:
        rng = Rng(int(case[5:]))
        sp = random_scene(rng, 30, True)
        cam = random_scene_camera(rng)
        lw = rng.uniform(-1.0, 1.0, (3, cam.height, cam.width))
        dw = rng.uniform(-1.0, 1.0, (cam.height, cam.width))
        ex = None
    f = orc.render_forward(sp, cam, keep_ctx=True)
    g = orc.render_backward(f, sp, cam, lw, dw, ex)
    tg = torch_ref.gradients(sp, cam, lw, dw, ex)
    for k in ("mean", "scale", "rotation", "falloff", "parent_falloff", "t", "sh"):
        scale = float(np.abs(tg[k]).max()) + 1e-12
        assert np.abs(g[k].astype(np.float64) - tg[k]).max() <= 1e-4 * scale, k


def test_oracle_band0_closed_form():  # test_render.cpp:556-576
    cam = axis_camera(48, 48, 70.0)
    sh = np.zeros((1, 48), np.float32)
    sh[0, :3] = 1.0
    sp = hs.RenderSplats.plain(np.array([[0, 0, 6]], np.float32), np.full((1, 3), 0.4, np.float32),
                               np.array([[1, 0, 0, 0]], np.float32), sh, np.array([0.5], np.float32))
    f = orc.render_forward(sp, cam, keep_ctx=True)
    n = 48.0 * 48.0 * 3.0
    g = orc.render_backward(f, sp, cam, np.full((3, 48, 48), 1.0 / n, np.float32))
    _, _, T, _ = f.images()
    mass = float((1.0 - T.astype(np.float64)).sum())
    for ch in range(3):
        assert g["sh"][0, ch] == pytest.approx(0.28209479177387814 * mass / n, rel=1e-4)


def test_oracle_exposure_gradient_outer_products():  # test_render.cpp:578-596
    rng = Rng(76)
    sp = random_scene(rng, 40, False)
    cam = random_scene_camera(rng)
    f = orc.render_forward(sp, cam, keep_ctx=True)
    lg = rng.uniform(-1.0, 1.0, (3, cam.height, cam.width))
    g = orc.render_backward(f, sp, cam, lg)
    c, _, _, _ = f.images()
    want = np.zeros((3, 4), np.float64)
    want[:, :3] = lg.reshape(3, -1).astype(np.float64) @ c.reshape(3, -1).astype(np.float64).T
    want[:, 3] = lg.reshape(3, -1).sum(1)
    assert np.allclose(g["exposure"], want, atol=1e-3)


def test_oracle_saturated_alpha_freezes_falloff():  # test_render.cpp:598-610
    cam = axis_camera(32, 32, 60.0)
    sp = gray_splat([0, 0, 4], 0.5, 1e5)
    f = orc.render_forward(sp, cam, keep_ctx=True)
    g = orc.render_backward(f, sp, cam, np.ones((3, 32, 32), np.float32))
    assert g["falloff"][0] == 0.0
    assert g["sh"][0, 0] != 0.0
    assert np.all(g["mean2d"][0] == 0.0)


def test_oracle_backward_needs_forward_state():
    sp = gray_splat([0, 0, 4], 0.5, 0.5)
    f = orc.render_forward(sp, axis_camera(16, 16, 30.0), keep_ctx=False)
    with pytest.raises(orc.OracleError):
        orc.render_backward(f, sp, axis_camera(16, 16, 30.0), np.ones((3, 16, 16), np.float32))


def _close(a, b, rtol, atol):
    """|a - b| <= atol + rtol * max(|a|, |b|), elementwise (tolerance for reordered float sums)."""
    return np.all(np.abs(a - b) <= atol + rtol * np.maximum(np.abs(a), np.abs(b)))


@pytest.mark.gpu
@pytest.mark.parametrize("seed,transitions", [(77, True), (78, False), (79, True)])
def test_gpu_backward_matches_oracle(renderer, seed, transitions):
    rng = Rng(seed)
    sp = random_scene(rng, 90, transitions)
    cam = random_scene_camera(rng)
    lg = rng.uniform(-1.0, 1.0, (3, cam.height, cam.width))
    dg = rng.uniform(-1.0, 1.0, (cam.height, cam.width))
    f = orc.render_forward(sp, cam, keep_ctx=True)
    want = orc.render_backward(f, sp, cam, lg, dg, EXPO)
    renderer.render_forward(sp, cam)
    got = renderer.render_backward(lg, dg, EXPO)
    for k in GRAD_KEYS:
        scale = float(np.abs(want[k]).max()) + 1e-12
        assert _close(got[k], want[k], 2e-3, 1e-4 * scale), k
    assert _close(got["exposure"], want["exposure"], 1e-4, 1e-3)


@pytest.mark.gpu
def test_gpu_backward_deterministic_and_band0(renderer):
    cam = axis_camera(48, 48, 70.0)
    sh = np.zeros((1, 48), np.float32)
    sh[0, :3] = 1.0
    sp = hs.RenderSplats.plain(np.array([[0, 0, 6]], np.float32), np.full((1, 3), 0.4, np.float32),
                               np.array([[1, 0, 0, 0]], np.float32), sh, np.array([0.5], np.float32))
    out = renderer.render_forward(sp, cam)
    n = 48.0 * 48.0 * 3.0
    g = renderer.render_backward(np.full((3, 48, 48), 1.0 / n, np.float32))
    mass = float((1.0 - out.transmittance.astype(np.float64)).sum())
    assert g["sh"][0, 0] == pytest.approx(0.28209479177387814 * mass / n, rel=1e-4)
    rng = Rng(80)
    sp = random_scene(rng, 120, True)
    cam = random_scene_camera(rng)
    lg = rng.uniform(-1.0, 1.0, (3, cam.height, cam.width))
    renderer.render_forward(sp, cam)
    g1 = renderer.render_backward(lg)
    g2 = renderer.render_backward(lg)
    for k in GRAD_KEYS + ("exposure",):
        assert np.array_equal(g1[k].view(np.uint32), g2[k].view(np.uint32)), k


@pytest.mark.gpu
def test_gpu_backward_hierarchy_frame_c1(renderer):
    """Backward over a render_hierarchy frame (C1: 100K leaves, 640x480): gradients w.r.t.
    the cut's interpolated splats, against the oracle over cut_render_splats."""
    from paper_2406_12080_b200 import scenes
    cfg = scenes.CONFIGS["c1"]
    h = scenes.hierarchy(cfg)
    cam = scenes.camera(cfg, 250)
    rng = Rng(91)
    lg = rng.uniform(-1.0, 1.0, (3, cam.height, cam.width))
    dg = rng.uniform(-1.0, 1.0, (cam.height, cam.width))
    out, cut = renderer.render_hierarchy(h, cam, cfg.tau, return_cut=True)
    got = renderer.render_backward(lg, dg, EXPO)
    oh = orc.OracleHierarchy(h)
    sp = orc.cut_render_splats(oh, cut.node, cut.t, cut.alpha_prime)
    f = orc.render_forward(sp, cam, keep_ctx=True)
    want = orc.render_backward(f, sp, cam, lg, dg, EXPO)
    assert got["mean"].shape[0] == len(cut)
    for k in GRAD_KEYS:
        scale = float(np.abs(want[k]).max()) + 1e-12
        assert _close(got[k], want[k], 5e-3, 1e-4 * scale), k


@pytest.mark.gpu
def test_gpu_backward_errors_and_empty(renderer):
    cam = axis_camera(32, 24, 40.0)
    renderer.render_forward(gray_splat([0, 0, -4], 0.5, 0.5), cam)  # behind the camera: culled
    g = renderer.render_backward(np.ones((3, 24, 32), np.float32))
    assert np.all(g["mean"] == 0) and np.all(g["sh"] == 0)
    assert g["exposure"][0, 3] == pytest.approx(24 * 32)  # sum of the loss gradient
    with pytest.raises(hs.Error):
        renderer.render_backward(np.ones((3, 10, 10), np.float32))  # DimensionMismatch
    with pytest.raises(hs.Error):
        renderer.render_backward(np.ones((3, 24, 32), np.float32), np.ones((5, 5), np.float32))


@pytest.mark.gpu
def test_gpu_backward_rejects_reselected_cut(renderer):
    """A hierarchy frame's backward re-assembles the splats from its cut: once the cut
    object holds another selection (select_cut on the same renderer), the frame's
    forward state is gone and backward reports MissingForwardState instead of
    differentiating the wrong cut."""
    from paper_2406_12080_b200 import scenes
    cfg = scenes.CONFIGS["c1"]
    h = scenes.hierarchy(cfg)
    lg = np.ones((3, cfg.height, cfg.width), np.float32)
    renderer.render_hierarchy(h, scenes.camera(cfg, 10), cfg.tau)
    renderer.render_backward(lg)  # fine: the cut is the one rendered
    renderer.select_cut(h, scenes.camera(cfg, 400), 0.5 * cfg.tau)  # a larger, different cut
    with pytest.raises(hs.Error) as e:
        renderer.render_backward(lg)
    assert e.value.code == hs.Errc.MissingForwardState
