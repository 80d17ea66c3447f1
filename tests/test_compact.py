"""compact (build.hpp:168-272): the multi-camera cut-union pass that removes
interior nodes no probed cut uses.  CPU: the oracle restatement against the
reference's own compaction tests (tests/test_build.cpp:199-236,
tests/acceptance.cpp:434-478).  GPU: hs_hierarchy_compact bit-exact (node for
node) against the oracle, and cut coverage preserved at every probed tau."""
import numpy as np
import pytest

import paper_2406_12080_b200 as hs
from oracle import oracle as orc
from paper_2406_12080_b200 import scenes
from tests.fixtures import Rng, random_gaussians

FIELDS = ("parent", "first_child", "child_count", "bmin", "bmax", "mean", "scale", "rot_wxyz", "falloff", "sh")


def _h(d):
    return hs.Hierarchy(*(d[f] for f in FIELDS))


def _leaf_partition(h, node):
    """cut_leaf_partition (tests/test_build.cpp): sorted leaf-mean keys under each cut node."""
    out = []
    for nd in node:
        stack, leaves = [int(nd)], []
        while stack:
            i = stack.pop()
            if h.child_count[i] == 0:
                leaves.append(tuple(h.mean[i]))
            else:
                stack.extend(range(int(h.first_child[i]), int(h.first_child[i] + h.child_count[i])))
        out.append(tuple(sorted(leaves)))
    return sorted(out)


def _ring_cams(n, radius, w, h, f, y=5.0):
    return [hs.look_at_camera([radius * np.cos(2.1 * i), y, radius * np.sin(2.1 * i)], [0, 0, 0], w, h, f)
            for i in range(n)]


def test_oracle_compaction_keeps_leaves_and_cut_coverage():  # test_build.cpp:199-227
    rng = Rng(54)
    h = hs.build_bvh(*random_gaussians(rng, 220, 6.0, 0.05, 0.3, 0.3, 0.9))
    cams = _ring_cams(3, 18.0, 256, 192, 300.0)
    oh = orc.OracleHierarchy(h)
    c = _h(orc.compact(oh, cams, 3.0))
    hs.validate_hierarchy(c)
    assert c.n <= h.n and c.leaf_count() == h.leaf_count()
    assert np.all(c.child_count[c.child_count > 0] >= 2)
    oc = orc.OracleHierarchy(c)
    tau = 3.0
    while tau <= 0.5 * 256.0:
        for cam in cams:
            before = _leaf_partition(h, orc.select_cut(oh, cam, tau)[0])
            after = _leaf_partition(c, orc.select_cut(oc, cam, tau)[0])
            assert before == after
        tau *= 2.0


def test_oracle_compaction_single_leaf_identity():  # test_build.cpp:229-236
    h = hs.build_bvh(np.zeros((1, 3)), np.full((1, 3), 0.1), [[1, 0, 0, 0]], [0.7], np.zeros((1, 48)))
    c = orc.compact(orc.OracleHierarchy(h), [hs.look_at_camera([0, 0, -5], [0, 0, 0], 64, 64, 100.0)])
    assert len(c["parent"]) == 1


def test_oracle_compaction_errors():
    h = hs.synth_city(300, seed=2)
    oh = orc.OracleHierarchy(h)
    with pytest.raises(orc.OracleError):
        orc.compact(oh, [], 3.0)
    with pytest.raises(orc.OracleError):
        orc.compact(oh, _ring_cams(1, 30.0, 64, 64, 60.0), 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("leaves,ncams,tau_min,tau_max", [(220, 3, 3.0, 0.0), (3000, 6, 3.0, 48.0),
                                                         (20000, 12, 1.5, 0.0), (1, 1, 3.0, 0.0)])
def test_gpu_compact_bit_exact(renderer, leaves, ncams, tau_min, tau_max):
    h = hs.synth_city(leaves, seed=leaves) if leaves > 1 else hs.build_bvh(
        np.zeros((1, 3)), np.full((1, 3), 0.1), [[1, 0, 0, 0]], [0.7], np.zeros((1, 48)))
    side = hs.scene_side(max(leaves, 21))
    cams = _ring_cams(ncams, 0.8 * side + 10.0, 320, 240, 250.0, y=0.3 * side + 4.0)
    want = orc.compact(orc.OracleHierarchy(h), cams, tau_min, tau_max)
    dc = renderer.compact(h, cams, tau_min, tau_max)
    got = renderer.download(dc)
    for f in FIELDS:
        assert np.array_equal(getattr(got, f).view(np.uint32), want[f].view(np.uint32)), f
    assert dc.leaf_count() == h.leaf_count()


@pytest.mark.gpu
def test_gpu_compact_preserves_cut_coverage(renderer):
    cfg = scenes.CONFIGS["c1"]
    h = scenes.hierarchy(cfg)
    cams = scenes.trajectory(cfg, 8, first=0)[::2]
    dc = renderer.compact(h, cams, 3.0, 48.0)
    c = renderer.download(dc)
    assert c.n < h.n and c.leaf_count() == h.leaf_count()
    hs.validate_hierarchy(c)
    dh = renderer.upload(h)
    tau = 3.0
    while tau <= 48.0:
        for cam in cams[:2]:
            a = renderer.select_cut(dh, cam, tau).node
            b = renderer.select_cut(dc, cam, tau).node
            assert _leaf_partition(h, a) == _leaf_partition(c, b)
        tau *= 2.0


@pytest.mark.gpu
def test_gpu_compact_edge_cases(renderer):
    """tau_max below tau_min (no probed level: only the breadth-first relayout), a single
    camera far away (coarse cuts), and the reference's argument checks."""
    h = hs.synth_city(2000, seed=5)
    cams = _ring_cams(2, 60.0, 128, 96, 120.0, y=20.0)
    oh = orc.OracleHierarchy(h)
    for tmin, tmax in ((3.0, 1.0), (50.0, 0.0), (3.0, 3.0)):
        want = orc.compact(oh, cams, tmin, tmax)
        got = renderer.download(renderer.compact(h, cams, tmin, tmax))
        for f in FIELDS:
            assert np.array_equal(getattr(got, f).view(np.uint32), want[f].view(np.uint32)), (tmin, tmax, f)
    with pytest.raises(hs.Error):
        renderer.compact(h, [], 3.0)
    with pytest.raises(hs.Error):
        renderer.compact(h, cams, 0.0)
