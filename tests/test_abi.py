"""C-ABI surface (CPU): the library loads, exports every entry point
include/hsplat_b200.h declares, and its host-side tools (synthetic hierarchy,
.h3dg IO, validation, build_bvh) behave like the reference's.  No device calls."""
import copy
import os
import re

import numpy as np
import pytest

import paper_2406_12080_b200 as hs
from paper_2406_12080_b200 import _native as N
from tests.fixtures import Rng, random_gaussians

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hsplat_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = N.lib()
    names = declared_symbols()
    assert len(names) >= 30
    for name in names:
        assert hasattr(L, name), name
        assert name in N._SIGS, f"{name} missing from the ctypes binding"


def test_status_names_follow_errc():
    L = N.lib()
    assert L.hs_status_name(0) == b"Ok"
    for e in hs.Errc:
        assert L.hs_status_name(int(e) + 1).decode() == e.name
    assert L.hs_status_name(100) == b"CudaError"


def test_context_without_device_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(hs.Error):
        hs.Renderer(0)


def test_synthetic_city_is_a_valid_build_bvh_tree():
    h = hs.synth_city(5000, seed=4)
    assert h.n == 9999 and h.leaf_count() == 5000
    hs.validate_hierarchy(h)
    # build_bvh layout: sibling pairs contiguous, parent < child (build.hpp:71-72)
    inner = np.flatnonzero(h.child_count > 0)
    assert np.all(h.child_count[inner] == 2)
    assert np.all(h.first_child[inner] > inner)
    assert np.all(h.parent[1:] < np.arange(1, h.n))
    q = np.linalg.norm(h.rot_wxyz, axis=1)
    assert np.all(np.abs(q - 1) < 1e-3)
    # deterministic
    h2 = hs.synth_city(5000, seed=4)
    assert np.array_equal(h.bmin, h2.bmin) and np.array_equal(h.sh, h2.sh)


def test_build_bvh_rejects_bad_leaves():
    with pytest.raises(hs.Error):
        hs.build_bvh(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0), np.zeros((0, 48)))
    rng = Rng(5)
    m, s, r, f, sh = random_gaussians(rng, 4)
    f[1] = 1.5  # leaf falloff must be in (0, 1] (build.hpp:77-78)
    with pytest.raises(hs.Error):
        hs.build_bvh(m, s, r, f, sh)


def test_h3dg_roundtrip(tmp_path):
    h = hs.synth_city(777, seed=9)
    p = str(tmp_path / "t.h3dg")
    hs.write_hierarchy(p, h)
    assert os.path.getsize(p) == 20 + 272 * h.n  # io.hpp:342-346
    g = hs.read_hierarchy(p)
    for f in ("parent", "first_child", "child_count", "bmin", "bmax", "mean", "scale", "rot_wxyz", "falloff", "sh"):
        assert np.array_equal(getattr(g, f), getattr(h, f)), f


def test_h3dg_corruption_errors(tmp_path):  # test_io.cpp corrupted-file cases
    h = hs.synth_city(50, seed=1)
    p = str(tmp_path / "t.h3dg")
    hs.write_hierarchy(p, h)
    raw = open(p, "rb").read()
    bad = tmp_path / "bad.h3dg"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(hs.Error) as e:
        hs.read_hierarchy(str(bad))
    assert e.value.code == hs.Errc.MalformedHeader
    bad.write_bytes(raw[:-5])
    with pytest.raises(hs.Error) as e:
        hs.read_hierarchy(str(bad))
    assert e.value.code == hs.Errc.TruncatedRecord
    b = bytearray(raw)
    b[16] = 4  # SH degree 4
    bad.write_bytes(bytes(b))
    with pytest.raises(hs.Error) as e:
        hs.read_hierarchy(str(bad))
    assert e.value.code == hs.Errc.UnsupportedShDegree
    with pytest.raises(hs.Error) as e:
        hs.read_hierarchy(str(tmp_path / "missing.h3dg"))
    assert e.value.code == hs.Errc.IoFailure


def test_validate_hierarchy_errors():  # model.hpp:118-139
    h = hs.synth_city(40, seed=2)
    g = copy.deepcopy(h)
    g.parent[0] = 1
    with pytest.raises(hs.Error, match="root"):
        hs.validate_hierarchy(g)
    g = copy.deepcopy(h)
    c = int(g.first_child[0])
    g.bmax[c, 0] = g.bmax[0, 0] + 1.0
    with pytest.raises(hs.Error, match="contain"):
        hs.validate_hierarchy(g)
    g = copy.deepcopy(h)
    g.rot_wxyz[3] *= 2
    with pytest.raises(hs.Error, match="unit quaternion"):
        hs.validate_hierarchy(g)
    g = copy.deepcopy(h)
    g.scale[5, 1] = 0
    with pytest.raises(hs.Error, match="scale"):
        hs.validate_hierarchy(g)


def test_camera_text_io(tmp_path):  # io.hpp:410-511
    cams = [hs.look_at_camera([1, 2, -5], [0, 0, 0], 64, 48, 70.0), hs.look_at_camera([0, 9, 3], [1, 0, 0], 80, 40, 50.0)]
    p = str(tmp_path / "cams.txt")
    hs.write_cameras(p, cams)
    back = hs.read_cameras(p)
    for a, b in zip(cams, back):
        assert (a.width, a.height) == (b.width, b.height)
        np.testing.assert_allclose(a.world_to_camera, b.world_to_camera, rtol=1e-6, atol=1e-7)
    pp = str(tmp_path / "path.txt")
    hs.write_camera_path(pp, [0.0, 1 / 30], cams)
    ts, c2 = hs.read_camera_path(pp)
    assert len(c2) == 2 and ts[1] > ts[0]
    with pytest.raises(hs.Error):
        hs.write_camera_path(pp, [1.0, 1.0], cams)
    (tmp_path / "bad.txt").write_text("64 48 70 70 32\n")
    with pytest.raises(hs.Error) as e:
        hs.read_cameras(str(tmp_path / "bad.txt"))
    assert e.value.code == hs.Errc.MalformedHeader
