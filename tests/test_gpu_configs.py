"""Parity at the BASELINE configs' other sensor shapes:

* C3 -- KITTI-shaped HDL-64, 64x2048 ``synthetic_intrinsics`` (the r0 = 0
  projection path), street scene, ICP + TSDF at 10 cm + marching cubes;
* C5 -- OS-128, 128x2048, r0 = 0.05 m, TSDF at 3 cm.

The golden vectors (tests/golden) pin the oracle to the reference at the
other shapes; here the CUDA path is checked against that pinned oracle on
these shapes, bit for bit where the arithmetic allows (float64-evaluated
transcendentals on both sides, RK_MATH_CR / math="cr").
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rk():
    import paper_2112_02779_b200 as rk
    return rk


def _case(name):
    from oracle import sensor as osens
    from oracle import synth as osynth
    from paper_2112_02779_b200 import scenes
    intr = scenes.hdl64() if name == "c3" else scenes.os128()
    S = osens.Sensor.from_intrinsics(intr)
    street = scenes.street_scene()
    gt = scenes.perturbation_pose(np.random.default_rng(1), 2.0, 0.3)
    dst = osynth.render(S, street)
    src = osynth.render(S, street, gt.R, gt.t)
    return intr, S, src, dst, gt


@pytest.fixture(scope="module", params=("c3", "c5"))
def case(request):
    return (request.param,) + _case(request.param)


def test_normals_bitexact(rk, case):
    from oracle import image as oimg
    name, intr, S, src, dst, gt = case
    nm = rk.compute_normal_map(rk.RangeImage(dst, intr))
    vec, valid = oimg.normals_cross(S, dst)
    assert np.array_equal(nm.valid, valid) and np.array_equal(nm.vectors, vec)


def test_register_cr_vs_oracle(rk, case):
    from oracle import icp as oicp
    from oracle import image as oimg
    from paper_2112_02779_b200 import lidar_model as lm
    name, intr, S, src, dst, gt = case
    vec, valid = oimg.normals_cross(S, dst)
    ref = oicp.register(S, src, dst, vec, valid, math="cr", fma="exact")
    with lm.math_mode(lm.MATH_CR):
        res = rk.register(rk.RangeImage(src, intr), rk.RangeImage(dst, intr))
    assert res.converged == ref["converged"]
    assert np.abs(res.pose.R - ref["R"]).max() < 1e-6 and np.abs(res.pose.t - ref["t"]).max() < 1e-6
    assert [(s.stride, s.iteration) for s in res.stats] == [(int(s[0]), int(s[1])) for s in ref["stats"]]
    # and the product math recovers the same pose within the north-star tolerance
    fast = rk.register(rk.RangeImage(src, intr), rk.RangeImage(dst, intr))
    assert np.abs(fast.pose.R - ref["R"]).max() < 1e-5 and np.abs(fast.pose.t - ref["t"]).max() < 1e-5


def test_tsdf_frame_cr_bitexact(rk, case):
    """One street frame into a fresh grid at the config's voxel size (C3 10 cm,
    C5 3 cm): key set, update count and every {tsdf, weight} bit-exact."""
    from oracle import tsdf as otsdf
    from paper_2112_02779_b200 import lidar_model as lm
    name, intr, S, src, dst, gt = case
    voxel = 0.10 if name == "c3" else 0.03
    og = {}
    keys, n_ref = otsdf.integrate_cloud_frame(og, S, dst, gt.R, gt.t, voxel, 4 * voxel,
                                              clip_max=30.0, math="cr")
    grid = rk.VoxelBlockGrid(voxel_size=voxel)
    with lm.math_mode(lm.MATH_CR):
        n = rk.integrate_cloud_frame(grid, rk.RangeImage(dst, intr), gt, clip_max=30.0)
    assert n == n_ref
    k, vox = grid.export_blocks()
    assert [tuple(x) for x in k.tolist()] == sorted(og)
    ref = np.stack([np.stack([og[t][0].reshape(-1), og[t][1].reshape(-1)], -1) for t in sorted(og)])
    assert np.array_equal(vox, ref)


def test_mesh_c3_vs_oracle(rk):
    """C3's marching cubes at 10 cm: the same vertex positions (exact) and the
    same triangles up to relabelling as the sequential oracle."""
    from oracle import mesh as omesh
    from oracle import tsdf as otsdf
    from paper_2112_02779_b200 import lidar_model as lm
    intr, S, src, dst, gt = _case("c3")
    og = {}
    otsdf.integrate_cloud_frame(og, S, dst, np.eye(3), np.zeros(3), 0.1, 0.4, clip_max=30.0, math="cr")
    V, T, N = omesh.extract_mesh(og, 0.1)
    grid = rk.VoxelBlockGrid(voxel_size=0.1)
    with lm.math_mode(lm.MATH_CR):
        rk.integrate_cloud_frame(grid, rk.RangeImage(dst, intr), rk.RigidTransform.identity(),
                                 clip_max=30.0)
    m = rk.extract_mesh(grid)
    assert m.n_vertices == V.shape[0] and m.n_triangles == T.shape[0] > 1000
    pos = {tuple(p): i for i, p in enumerate(V.tolist())}
    remap = np.array([pos[tuple(p)] for p in m.vertices.tolist()])
    assert np.abs(m.normals - N[remap]).max() < 1e-9
    canon = lambda tris: {tuple(np.roll(t, -int(np.argmin(t)))) for t in tris.tolist()}  # noqa: E731
    assert canon(remap[m.triangles]) == canon(T)
