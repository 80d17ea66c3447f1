"""Multi-chunk scenes (BASELINE config[4]): chunk + skybox
generation, consolidate's breadth-first serialisation (scene.hpp:281-316)
restated in numpy (oracle.consolidate_bfs), and the device assembly
(hs_hierarchy_assemble) checked node for node against it; the assembled
hierarchy then renders bit-exactly like the oracle."""
import numpy as np
import pytest

import paper_2406_12080_b200 as hs
from oracle import oracle as orc
from paper_2406_12080_b200 import scenes

FIELDS = ("parent", "first_child", "child_count", "bmin", "bmax", "mean", "scale", "rot_wxyz", "falloff", "sh")


def _as_hierarchy(d):
    return hs.Hierarchy(*(d[f] for f in FIELDS))


def test_chunk_parts_tile_the_scene():
    parts = list(scenes.chunk_parts(4 * 2100, grid=2, sky=300, seed=5))
    assert [n for n, _ in parts] == ["chunk_0_0", "chunk_1_0", "chunk_0_1", "chunk_1_1", "skybox"]
    side = hs.scene_side(2100)
    for name, h in parts[:4]:
        ix, iz = int(name[6]), int(name[8])
        leaf = h.child_count == 0
        c = h.mean[leaf].mean(axis=0)
        assert abs(c[0] - (ix - 0.5) * side) < 0.2 * side and abs(c[2] - (iz - 0.5) * side) < 0.2 * side
        hs.validate_hierarchy(h)
    sky = parts[4][1]
    hs.validate_hierarchy(sky)
    r = np.linalg.norm(sky.mean[sky.child_count == 0], axis=1)
    assert np.allclose(r, 5.0 * 2 * side * np.sqrt(2.0), rtol=1e-5)  # make_skybox shell radius
    assert np.all(sky.sh == 0.0) and np.all(sky.falloff[sky.child_count == 0] == 0.7)


def test_consolidate_bfs_single_part_is_valid_bfs():
    h = hs.synth_city(3000, seed=9)
    d = orc.consolidate_bfs([h])
    b = _as_hierarchy(d)
    hs.validate_hierarchy(b)
    assert b.n == h.n and b.leaf_count() == h.leaf_count()
    idx = np.arange(1, b.n)
    assert np.all(b.parent[idx] < idx)  # parent < child
    # depth is non-decreasing along the serialisation (breadth first)
    depth = np.zeros(b.n, np.int64)
    for i in range(1, b.n):
        depth[i] = depth[b.parent[i]] + 1
    assert np.all(np.diff(depth) >= 0)
    # the same Gaussians, permuted
    assert np.array_equal(np.sort(b.mean[:, 0]), np.sort(h.mean[:, 0]))


@pytest.mark.gpu
@pytest.mark.parametrize("grid,sky", [(1, 0), (2, 400), (3, 0)])
def test_device_assembly_matches_bfs_oracle(renderer, grid, sky):
    parts = [h for _, h in scenes.chunk_parts(grid * grid * 1500, grid=grid, sky=sky, seed=3)]
    dh = renderer.assemble(parts)
    got = renderer.download(dh)
    k = len(parts)
    root = None
    if k > 1:
        root = {f: getattr(got, f)[0] for f in ("bmin", "bmax", "mean", "scale", "rot_wxyz", "falloff", "sh")}
        root["kid_scale"], root["kid_rot"] = got.scale[1:1 + k], got.rot_wxyz[1:1 + k]
        # root box = union of the part boxes; forest roots keep mean/falloff/SH
        assert np.array_equal(got.bmin[0], np.min([p.bmin[0] for p in parts], axis=0))
        assert np.array_equal(got.bmax[0], np.max([p.bmax[0] for p in parts], axis=0))
        for p in range(k):
            assert np.array_equal(got.mean[1 + p], parts[p].mean[0])
            assert np.array_equal(got.sh[1 + p], parts[p].sh[0])
    want = orc.consolidate_bfs(parts, root)
    for f in FIELDS:
        assert np.array_equal(getattr(got, f).view(np.uint32), want[f].view(np.uint32)), f
    hs.validate_hierarchy(got)
    assert dh.leaf_count() == sum(p.leaf_count() for p in parts)


@pytest.mark.gpu
def test_multichunk_render_bit_exact(renderer):
    cfg = scenes.Config("mc", 16 * 2000, 320, 240, 200.0, 3.0, altitude=20.0, standoff=15.0, lookahead=80.0)
    dh = scenes.multichunk(renderer, cfg.leaves, grid=4, sky=1000, seed=2)
    host = renderer.download(dh)
    oh = orc.OracleHierarchy(host)
    for frame in (0, 130, 620):
        cam = scenes.camera(cfg, frame)
        out, cut = renderer.render_hierarchy(dh, cam, cfg.tau, return_cut=True)
        f = orc.render_hierarchy(oh, cam, cfg.tau, keep_ctx=False)
        node, t, a = f.cut()
        assert np.array_equal(cut.node, node)
        assert np.array_equal(cut.alpha_prime.view(np.uint32), a.view(np.uint32))
        c, d, T, rc = f.images()
        assert np.array_equal(out.color.view(np.uint32), c.view(np.uint32))
        assert np.array_equal(out.transmittance.view(np.uint32), T.view(np.uint32))
        assert out.rendered_count == rc


@pytest.mark.gpu
def test_assemble_errors(renderer):
    with pytest.raises(hs.Error):
        renderer.assemble([])
    parts = [hs.synth_city(300, seed=s) for s in range(65)]
    with pytest.raises(hs.Error):
        renderer.assemble(parts)  # more than 64 parts
