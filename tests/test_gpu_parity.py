"""Parity of the CUDA path (librkb200.so, via the package API / C ABI) with the
reference's golden vectors and with the CPU oracle.

Contract (BASELINE.json north_star):
* bit-exact: sensor tables, row lookup, pyramid indices and point clouds,
  normals, voxel-block allocation; with RK_MATH_CR (float64-evaluated
  transcendentals in both kernel and oracle) also projection, association
  sets and TSDF values;
* with the opt-in RK_MATH_FAST (minimax atan2/asin, MUFU square roots,
  float32 ICP move, vs numpy's SVML): >= 99.9 % correspondence-mask
  agreement, poses within 1e-5 rad / 1e-5 m with equal iteration counts,
  TSDF values within 1e-5 (the "*_vs_reference" tests that use the
  fast_math fixture).  The default RK_MATH_NP is bit-exact against the
  reference: tests/test_gpu_numpy_exact.py.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PAIRS = ("room", "street", "synth")
SENSOR_OF = {"room": "small", "street": "ouster", "synth": "synth"}


@pytest.fixture(scope="module")
def rk():
    import paper_2112_02779_b200 as rk
    return rk


def rot_err(Ra, Rb):
    c = (np.trace(Ra.T @ Rb) - 1.0) / 2.0
    return float(np.arccos(np.clip(c, -1.0, 1.0)))


def set_agreement(a, b):
    a, b = set(map(int, a)), set(map(int, b))
    if not a and not b:
        return 1.0
    return len(a & b) / len(a | b)


# ---------------------------------------------------------------- sensor model

def _ulps(a, b):
    """float32 ulp distance (same-sign finite values)."""
    ia = a.astype(np.float32).view(np.int32).astype(np.int64)
    ib = b.astype(np.float32).view(np.int32).astype(np.int64)
    return np.abs(ia - ib)


def test_fast_math_ulp(rk, sensors):
    """RK_MATH_FAST's projection against float64-evaluated transcendentals
    (RK_MATH_CR): azimuth/elevation within a few ulp, i.e. the same
    accuracy class as numpy's SVML float32 arctan2/arcsin (<= 3 ulp)."""
    from paper_2112_02779_b200 import lidar_model as lm
    intr = sensors["ouster"]
    rng = np.random.default_rng(11)
    n = 400_000
    d = rng.normal(size=(n, 3))
    d[:, 2] *= 0.25
    pts = (d / np.linalg.norm(d, axis=1, keepdims=True) * rng.uniform(0.3, 60.0, (n, 1))).astype(np.float32)
    uf, vf, rf, sf = rk.project_many(pts, intr, single=True, refine=False, math=lm.MATH_FAST)
    uc, vc, rc, sc = rk.project_many(pts, intr, single=True, refine=False, math=lm.MATH_CR)
    ul, vl, rl, sl = rk.project_many(pts, intr, single=True, refine=False, math=lm.MATH_LIBM)
    ok = (sc == 0) & (sf == 0)
    assert np.mean(sf == sc) >= 0.9999 and np.mean(sl == sc) >= 0.9999
    assert np.mean(vf[ok] == vc[ok]) >= 0.9999
    # column: |du| bounded by a few ulp of the azimuth scaled into pixels
    du = np.abs(uf[ok].astype(np.float64) - uc[ok])
    du = np.minimum(du, intr.width - du)
    assert du.max() < 2e-3, du.max()
    assert np.mean(du == 0) >= 0.5
    assert np.array_equal(rf, rc)          # r has no transcendental: exact in every mode
    # FAST is no further from correctly rounded than CUDA's libm
    dl = np.abs(ul[ok].astype(np.float64) - uc[ok])
    dl = np.minimum(dl, intr.width - dl)
    assert du.mean() <= 2.0 * dl.mean() + 1e-6


@pytest.mark.parametrize("name", ("small", "synth", "ouster"))
def test_project_f32_cr_bitexact_vs_oracle(rk, name, sensors, osensors, golden_proj):
    from paper_2112_02779_b200.lidar_model import MATH_CR
    pts = golden_proj[f"{name}/p32_in"]
    u, v, r, st = rk.project_many(pts, sensors[name], single=True, math=MATH_CR)
    ou, ov, orr, ost = osensors[name].project_f32(pts, math="cr")
    ok = ost == 0
    assert np.array_equal(st, ost)
    assert np.array_equal(v[ok], ov[ok]) and np.array_equal(u[ok], ou[ok])
    assert np.array_equal(r, orr)


@pytest.mark.usefixtures("fast_math")
@pytest.mark.parametrize("name", ("small", "synth", "ouster"))
def test_project_f32_fast_vs_reference(rk, name, sensors, golden_proj):
    g = golden_proj
    pts = g[f"{name}/p32_in"]
    u, v, r, st = rk.project_many(pts, sensors[name], single=True)
    assert np.mean(st == g[f"{name}/p32_st"]) >= 0.999
    both = (st == 0) & (g[f"{name}/p32_st"] == 0)
    assert np.mean(v[both] == g[f"{name}/p32_v"][both]) >= 0.999
    assert np.array_equal(r, g[f"{name}/p32_r"])           # no transcendental on r
    du = np.abs(u[both] - g[f"{name}/p32_u"][both])
    du = np.minimum(du, sensors[name].width - du)
    assert np.percentile(du, 99.9) < 1e-3


@pytest.mark.parametrize("name", ("small", "synth", "ouster"))
def test_project_f64_vs_reference(rk, name, sensors, golden_proj):
    g = golden_proj
    u, v, r, st = rk.project_many(g[f"{name}/p64_in"], sensors[name])
    assert np.mean(st == g[f"{name}/p64_st"]) >= 0.999
    both = (st == 0) & (g[f"{name}/p64_st"] == 0)
    assert np.mean(v[both] == g[f"{name}/p64_v"][both]) >= 0.999
    same = both & (v == g[f"{name}/p64_v"])
    assert np.abs(u[same] - g[f"{name}/p64_u"][same]).max() < 1e-9
    assert np.abs(r - g[f"{name}/p64_r"]).max() < 1e-9


@pytest.mark.parametrize("name", ("small", "synth", "ouster"))
def test_rows_and_lookup_bitexact(rk, name, sensors, golden_proj):
    g, intr = golden_proj, sensors[name]
    assert np.array_equal(intr.row_from_elevation(g[f"{name}/phi64"]), g[f"{name}/row64"])
    assert np.array_equal(intr.row_from_elevation(g[f"{name}/phi32"]), g[f"{name}/row32"])
    assert np.array_equal(intr.inv_elevation_lut.lookup(g[f"{name}/phi64"]), g[f"{name}/lookup64"])


# ---------------------------------------------------------------- images (K1, K2)

@pytest.mark.parametrize("pair", PAIRS)
def test_normals_bitexact(rk, pair, sensors, golden_icp):
    img = rk.RangeImage(golden_icp[f"{pair}/dst"], sensors[SENSOR_OF[pair]])
    nm = rk.compute_normal_map(img)
    assert np.array_equal(nm.valid, golden_icp[f"{pair}/nvalid"])
    assert np.array_equal(nm.vectors, golden_icp[f"{pair}/nrm"])


@pytest.mark.parametrize("pair", ("room", "synth"))
def test_point_clouds_and_pyramid_bitexact(rk, pair, sensors, osensors, golden_icp):
    from oracle import image as oimg
    from paper_2112_02779_b200.range_image import points_at_stride, stride_indices
    intr = sensors[SENSOR_OF[pair]]
    img = rk.RangeImage(golden_icp[f"{pair}/src"], intr)
    assert np.array_equal(rk.to_point_cloud(img, 0.5, 20.0), golden_icp[f"{pair}/cloud"])
    for s in (1, 2, 4):
        assert np.array_equal(points_at_stride(img, s), golden_icp[f"{pair}/pts_s{s}"])
        idx, _ = stride_indices(img, s, 0.5, 20.0)
        v, u = oimg.stride_indices(golden_icp[f"{pair}/src"], s, 0.5, 20.0)
        assert np.array_equal(idx.cpu().numpy(), v * intr.width + u)


def test_pyramid_edge_cases(rk, sensors):
    from paper_2112_02779_b200.range_image import stride_indices
    intr = sensors["small"]
    empty = rk.RangeImage(np.zeros((intr.height, intr.width), np.float32), intr)
    for s in (1, 3, 4, 7):
        idx, _ = stride_indices(empty, s)
        assert idx.numel() == 0
    full = rk.RangeImage(np.full((intr.height, intr.width), 5.0, np.float32), intr)
    for s in (1, 3, 5, 33):
        idx, _ = stride_indices(full, s)
        Hs, Ws = -(-intr.height // s), -(-intr.width // s)
        assert idx.numel() == Hs * Ws
        vv, uu = np.meshgrid(np.arange(0, intr.height, s), np.arange(0, intr.width, s), indexing="ij")
        assert np.array_equal(idx.cpu().numpy(), (vv * intr.width + uu).reshape(-1))


# ---------------------------------------------------------------- association

def _src_cloud(rk, pair, sensors, golden_icp):
    return rk.to_point_cloud(rk.RangeImage(golden_icp[f"{pair}/src"], sensors[SENSOR_OF[pair]]))


@pytest.mark.parametrize("pair", PAIRS)
def test_correspondences_cr_bitexact_vs_oracle(rk, pair, sensors, osensors, golden_icp):
    from oracle import icp as oicp
    from paper_2112_02779_b200 import lidar_model as lm
    g, intr = golden_icp, sensors[SENSOR_OF[pair]]
    dst = rk.RangeImage(g[f"{pair}/dst"], intr)
    nm = rk.compute_normal_map(dst)
    src_pts = _src_cloud(rk, pair, sensors, golden_icp)
    M = g[f"{pair}/corr_pose"]
    pose = rk.RigidTransform(M[:3, :3], M[:3, 3])
    with lm.math_mode(lm.MATH_CR):
        for s in (1, 2, 4):
            c = rk.projective_correspondences(src_pts, dst, nm, pose, 0.5 * s, s, single=True)
            sel, tgt, nrm, _ = oicp.correspondences_f32(osensors[SENSOR_OF[pair]], src_pts, g[f"{pair}/dst"],
                                                        g[f"{pair}/nrm"], g[f"{pair}/nvalid"], M[:3, :3],
                                                        M[:3, 3], 0.5 * s, s, math="cr")
            assert np.array_equal(c.source, src_pts[sel])
            assert np.array_equal(c.target, tgt) and np.array_equal(c.normal, nrm)


@pytest.mark.usefixtures("fast_math")
@pytest.mark.parametrize("pair", PAIRS)
def test_correspondence_masks_vs_reference(rk, pair, sensors, golden_icp):
    g, intr = golden_icp, sensors[SENSOR_OF[pair]]
    dst = rk.RangeImage(g[f"{pair}/dst"], intr)
    nm = rk.compute_normal_map(dst)
    src_pts = _src_cloud(rk, pair, sensors, golden_icp)
    M = g[f"{pair}/corr_pose"]
    pose = rk.RigidTransform(M[:3, :3], M[:3, 3])
    index = {tuple(r): i for i, r in enumerate(src_pts.tolist())}
    for s in ((4,) if pair == "street" else (1, 2, 4)):
        c = rk.projective_correspondences(src_pts, dst, nm, pose, 0.5 * s, s, single=True)
        got = [index[tuple(r)] for r in c.source.tolist()]
        assert set_agreement(got, g[f"{pair}/c32_s{s}_sel"]) >= 0.999
    sub = src_pts[::7] if pair == "street" else src_pts[::2]
    c = rk.projective_correspondences(sub, dst, nm, pose, 0.5, 1)
    index = {tuple(r): i for i, r in enumerate(sub.tolist())}
    got = np.array([index[tuple(r)] for r in c.source.tolist()])
    assert set_agreement(got, g[f"{pair}/c64_sel"]) >= 0.999
    common, ia, ib = np.intersect1d(got, g[f"{pair}/c64_sel"], return_indices=True)
    assert np.abs(c.target[ia] - g[f"{pair}/c64_tgt"][ib]).max() < 1e-9


# ---------------------------------------------------------------- registration (K3)

@pytest.mark.usefixtures("fast_math")
@pytest.mark.parametrize("pair", PAIRS)
def test_register_vs_reference(rk, pair, sensors, golden_icp):
    g, intr = golden_icp, sensors[SENSOR_OF[pair]]
    src, dst = rk.RangeImage(g[f"{pair}/src"], intr), rk.RangeImage(g[f"{pair}/dst"], intr)
    res = rk.register(src, dst)
    M = g[f"{pair}/reg_pose"]
    stats = g[f"{pair}/reg_stats"]
    assert res.converged == bool(g[f"{pair}/reg_converged"])
    assert rot_err(res.pose.R, M[:3, :3]) < 1e-5
    assert np.linalg.norm(res.pose.t - M[:3, 3]) < 1e-5
    got = np.array([[s.stride, s.iteration, s.n_correspondences] for s in res.stats])
    assert got.shape[0] == stats.shape[0]                      # same iteration count per level
    assert np.array_equal(got[:, :2], stats[:, :2])
    assert np.all(np.abs(got[:, 2] - stats[:, 2]) <= np.maximum(2, 1e-3 * stats[:, 2]))
    cost = np.array([s.cost for s in res.stats])
    assert np.allclose(cost, stats[:, 3], rtol=1e-3)


@pytest.mark.parametrize("pair", PAIRS)
def test_register_cr_vs_oracle(rk, pair, sensors, osensors, golden_icp):
    from oracle import icp as oicp
    from paper_2112_02779_b200 import lidar_model as lm
    g, intr = golden_icp, sensors[SENSOR_OF[pair]]
    src, dst = rk.RangeImage(g[f"{pair}/src"], intr), rk.RangeImage(g[f"{pair}/dst"], intr)
    with lm.math_mode(lm.MATH_CR):
        res = rk.register(src, dst)
    ref = oicp.register(osensors[SENSOR_OF[pair]], g[f"{pair}/src"], g[f"{pair}/dst"], g[f"{pair}/nrm"],
                        g[f"{pair}/nvalid"], math="cr")
    assert res.converged == ref["converged"]
    assert rot_err(res.pose.R, ref["R"]) < 1e-6 and np.linalg.norm(res.pose.t - ref["t"]) < 1e-6
    assert [s.n_correspondences for s in res.stats] == [s[2] for s in ref["stats"]]


def test_register_batch_deterministic_and_consistent(rk, sensors, golden_icp):
    import torch
    from paper_2112_02779_b200.range_image import normals_cross_batch
    from paper_2112_02779_b200 import _native as nat
    from paper_2112_02779_b200.lidar_model import default_math
    g, intr = golden_icp, sensors["ouster"]
    # a batch inside register()'s latency tier (the 16-CTA clusters when the
    # device co-schedules several), so the per-thread split -- and every
    # bit -- matches the single call; other tiers: the 1e-5 tier test below
    cap16 = nat.load().rk_icp_cluster_capacity(default_math(), 16)
    B = min(8, cap16) if cap16 >= 2 else 8
    src = torch.from_numpy(g["street/src"]).cuda()[None].repeat(B, 1, 1)
    dst = torch.from_numpy(g["street/dst"]).cuda()[None].repeat(B, 1, 1)
    surf = normals_cross_batch(intr, dst)
    a = rk.register_batch(intr, src, dst, surf)
    b = rk.register_batch(intr, src, dst, surf)
    assert torch.equal(a.poses, b.poses)
    assert bool((a.poses == a.poses[:1]).all())
    single = rk.register(rk.RangeImage(g["street/src"], intr), rk.RangeImage(g["street/dst"], intr))
    assert np.array_equal(a.pose(0).matrix(), single.pose.matrix())


def test_register_batch_preallocated_outputs(rk, sensors, golden_icp):
    """register_batch(out=...) writes into the caller's tensors (the latency
    graph's packed buffer) with the same bits, and rejects wrong shapes."""
    import torch
    g, intr = golden_icp, sensors["ouster"]
    src = torch.from_numpy(g["street/src"]).cuda()[None]
    dst = torch.from_numpy(g["street/dst"]).cuda()[None]
    cfg = rk.RegistrationConfig()
    ref = rk.register_batch(intr, src, dst, config=cfg, with_stats=True)
    out = (torch.empty((1, 12), dtype=torch.float64, device="cuda"),
           torch.empty((1,), dtype=torch.int32, device="cuda"),
           torch.empty((1,), dtype=torch.int32, device="cuda"),
           torch.empty((1, cfg.max_iterations, 5), dtype=torch.float64, device="cuda"))
    res = rk.register_batch(intr, src, dst, config=cfg, with_stats=True, out=out)
    assert res.poses is out[0] and torch.equal(out[0], ref.poses)
    assert torch.equal(out[1], ref.status) and torch.equal(out[2], ref.iterations)
    n = int(ref.iterations[0])
    assert torch.equal(out[3][:, :n], ref.stats[:, :n])
    bad = (out[0].float(),) + out[1:]
    with pytest.raises(ValueError):
        rk.register_batch(intr, src, dst, config=cfg, with_stats=True, out=bad)


def test_register_batch_index_dtypes_and_validation(rk, sensors, golden_icp):
    """int64 pair indices (torch's default) give the same poses as int32 ones
    (the converted copies stay alive across the launch), and host-side or
    mis-shaped index / init tensors are rejected before any launch."""
    import torch
    g, intr = golden_icp, sensors["ouster"]
    src = torch.from_numpy(np.stack([g["street/src"], g["street/dst"]])).cuda()
    dst = torch.from_numpy(np.stack([g["street/dst"], g["street/src"]])).cuda()
    ps64 = torch.tensor([0, 1, 0, 1], dtype=torch.int64, device="cuda")
    pd64 = torch.tensor([0, 0, 1, 1], dtype=torch.int64, device="cuda")
    a = rk.register_batch(intr, src, dst, pair_src=ps64, pair_dst=pd64)
    b = rk.register_batch(intr, src, dst, pair_src=ps64.int(), pair_dst=pd64.int())
    assert torch.equal(a.poses, b.poses) and torch.equal(a.status, b.status)
    # pair 0 = (src 0, dst 0) is the golden street pair; pair 1 = (dst image, dst image)
    single = rk.register(rk.RangeImage(g["street/src"], intr), rk.RangeImage(g["street/dst"], intr))
    assert np.abs(a.pose(0).matrix() - single.pose.matrix()).max() < 1e-5
    assert np.abs(a.pose(1).matrix() - np.eye(4)).max() < 1e-6
    with pytest.raises(ValueError):
        rk.register_batch(intr, src, dst, pair_src=ps64.cpu(), pair_dst=pd64)
    with pytest.raises(ValueError):
        rk.register_batch(intr, src, dst, pair_src=ps64, pair_dst=pd64[:3])
    with pytest.raises(ValueError):
        rk.register_batch(intr, src, dst, pair_src=None, pair_dst=pd64)
    with pytest.raises(ValueError):
        rk.register_batch(intr, src, dst, pair_src=ps64, pair_dst=pd64,
                          inits=torch.zeros((3, 12), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        rk.register_batch(intr, src, dst, pair_src=ps64, pair_dst=pd64,
                          inits=torch.zeros((4, 12), dtype=torch.float64))


@pytest.mark.parametrize("batch", [1, 2, 7, 8, 9, 15, 16, 17, 18, 19, 33, 34, 37, 38, 74, 75, 148, 149, 300])
def test_register_batch_tiers_match_register(rk, sensors, golden_icp, batch):
    """The launcher picks a cluster size (x16/x8/x4/x2) or CTA width (1024/512/256; 512/256 in NP)
    from the batch size, which changes each pair's float32 per-thread split,
    so results may differ in the last bits between tiers (INTEGRATION.md,
    'Batch-size dependence').  Every tier stays inside the pose contract
    (1e-5) of the single-pair register() on the golden street pair, with
    the same per-pair iteration count."""
    import torch
    g, intr = golden_icp, sensors["ouster"]
    src = torch.from_numpy(g["street/src"]).cuda()[None]
    dst = torch.from_numpy(g["street/dst"]).cuda()[None]
    zeros = torch.zeros(batch, dtype=torch.int32, device="cuda")
    res = rk.register_batch(intr, src, dst, pair_src=zeros, pair_dst=zeros)
    single = rk.register(rk.RangeImage(g["street/src"], intr), rk.RangeImage(g["street/dst"], intr))
    P = res.poses.cpu().numpy()
    ref = single.pose.as_row12()
    assert np.abs(P - ref[None]).max() < 1e-5
    assert bool((res.poses == res.poses[:1]).all())      # one tier per launch: all pairs equal
    assert set(res.iterations.cpu().tolist()) == {len(single.stats)}


@pytest.mark.parametrize("pair", PAIRS)
def test_register_batch_surfel_pyramid_bitidentical(rk, pair, sensors, golden_icp):
    """Coarse levels gathering from the decimated surfel maps see exactly the
    values of the strided full-resolution reads: poses and iteration counts
    are bit-identical (also for a sensor whose view width is not a multiple
    of the CTA, i.e. the generic walk)."""
    import torch
    from paper_2112_02779_b200.range_image import SurfelPyramid, normals_cross_batch
    g, intr = golden_icp, sensors[SENSOR_OF[pair]]
    src = torch.from_numpy(g[f"{pair}/src"]).cuda()[None].repeat(3, 1, 1)
    dst = torch.from_numpy(g[f"{pair}/dst"]).cuda()[None].repeat(3, 1, 1)
    cfg = rk.RegistrationConfig(schedule=((4, 20), (3, 5), (2, 20), (1, 10)))
    flat = normals_cross_batch(intr, dst)
    pyr = normals_cross_batch(intr, dst, strides=[s for s, _ in cfg.schedule])
    assert isinstance(pyr, SurfelPyramid) and set(pyr.offsets) == {1, 2, 3, 4}
    HW = intr.height * intr.width
    assert torch.equal(pyr.data[:, :HW, :4].reshape(flat.shape), flat)
    if pyr.data.shape[-1] == 8:  # RK_SURFEL_REC=32 builds carry the target
        # the record's target is the reference's float32 r * dir32 + origin32 (registration.py:168-176)
        d32 = np.stack(intr.ray_tables_flat_f32[0], -1)
        o32 = np.stack(intr.ray_tables_flat_f32[1], -1)
        r = g[f"{pair}/dst"].reshape(-1).astype(np.float32)
        tgt = r[:, None] * d32 + o32[np.arange(HW) % intr.width]
        got = pyr.data[0, :HW, 4:7].cpu().numpy()
        assert np.array_equal(got[r > 0], tgt[r > 0])
    for s, off in pyr.offsets.items():  # decimated maps = the strided full map
        Hs, Ws = -(-intr.height // s), -(-intr.width // s)
        lvl = pyr.data[:, off:off + Hs * Ws, :4].reshape(3, Hs, Ws, 4)
        assert torch.equal(lvl, flat[:, ::s, ::s])
    a = rk.register_batch(intr, src, dst, flat, config=cfg, with_stats=True)
    b = rk.register_batch(intr, src, dst, pyr, config=cfg, with_stats=True)
    assert torch.equal(a.poses, b.poses) and torch.equal(a.iterations, b.iterations)
    n = int(a.iterations[0])
    assert torch.equal(a.stats[:, :n], b.stats[:, :n])
    with pytest.raises(ValueError):
        rk.register_batch(intr, src, dst, normals_cross_batch(intr, dst, strides=[4]), config=cfg)


@pytest.mark.parametrize("wpp", ("1", "8"))
def test_register_batch_layouts_match_reference(rk, wpp, sensors, golden_icp, monkeypatch):
    """Warp-per-pair and CTA-per-pair kernels both meet the reference contract."""
    import torch
    monkeypatch.setenv("RK_ICP_WPP", wpp)
    g, intr = golden_icp, sensors["ouster"]
    src = torch.from_numpy(g["street/src"]).cuda()[None].repeat(3, 1, 1)
    dst = torch.from_numpy(g["street/dst"]).cuda()[None].repeat(3, 1, 1)
    res = rk.register_batch(intr, src, dst, with_stats=True)
    M = g["street/reg_pose"]
    for b in range(3):
        assert int(res.status[b]) == 0
        assert int(res.iterations[b]) == g["street/reg_stats"].shape[0]
        P = res.pose(b)
        assert rot_err(P.R, M[:3, :3]) < 1e-5 and np.linalg.norm(P.t - M[:3, 3]) < 1e-5


@pytest.mark.parametrize("cluster", ("0", "2", "4", "8", "16"))
def test_register_latency_clusters_match_reference(rk, cluster, sensors, golden_icp, monkeypatch):
    """Latency mode: one pair per wide CTA (0) or per cluster of 2/4/8/16
    CTAs reducing through distributed shared memory -- same contract, and a
    bad pair index still yields its defined status on every cluster size."""
    import torch
    from paper_2112_02779_b200.registration import ICP_BAD_PAIR
    monkeypatch.setenv("RK_ICP_CLUSTER", cluster)
    g, intr = golden_icp, sensors["ouster"]
    src = torch.from_numpy(g["street/src"]).cuda()[None].repeat(2, 1, 1)
    dst = torch.from_numpy(g["street/dst"]).cuda()[None].repeat(2, 1, 1)
    ps = torch.tensor([0, 1, 5], dtype=torch.int32, device="cuda")
    res = rk.register_batch(intr, src, dst, pair_src=ps, pair_dst=torch.tensor([1, 0, 0], dtype=torch.int32,
                                                                                device="cuda"), with_stats=True)
    M = g["street/reg_pose"]
    st = g["street/reg_stats"]
    for b in range(2):
        assert int(res.status[b]) == 0
        assert int(res.iterations[b]) == st.shape[0]
        P = res.pose(b)
        assert rot_err(P.R, M[:3, :3]) < 1e-5 and np.linalg.norm(P.t - M[:3, 3]) < 1e-5
        got = res.stats[b, :st.shape[0]].cpu().numpy()
        assert np.array_equal(got[:, :2], st[:, :2])  # stride, iteration
        assert np.all(np.abs(got[:, 2] - st[:, 2]) <= np.maximum(2, 1e-3 * st[:, 2]))
    assert int(res.status[2]) == ICP_BAD_PAIR and int(res.iterations[2]) == 0


def test_register_nonconvergence_and_identity(rk, sensors, golden_icp):
    intr = sensors["synth"]
    img = rk.RangeImage(golden_icp["synth/dst"], intr)
    empty = rk.RangeImage(np.zeros((intr.height, intr.width), np.float32), intr)
    assert not rk.register(img, empty).converged
    res = rk.register(img, img)
    assert res.converged
    assert rot_err(res.pose.R, np.eye(3)) < 1e-6 and np.linalg.norm(res.pose.t) < 1e-6


def test_centroid_vs_reference(rk, sensors, golden_icp):
    for pair in PAIRS:
        intr = sensors[SENSOR_OF[pair]]
        s = rk.to_point_cloud(rk.RangeImage(golden_icp[f"{pair}/src"], intr))
        d = rk.to_point_cloud(rk.RangeImage(golden_icp[f"{pair}/dst"], intr))
        t = rk.initial_translation_by_centroids(s, d).t
        assert np.abs(t - golden_icp[f"{pair}/centroid_t"]).max() < 1e-12


def test_gauss_newton_f64_helpers(rk):
    from paper_2112_02779_b200 import registration as reg
    g = np.random.default_rng(8)
    p = g.normal(scale=3.0, size=(80, 3))
    q = p + g.normal(scale=0.05, size=(80, 3))
    n = g.normal(size=(80, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    corr = reg.CorrespondenceSet(p, q, n)
    xi, _ = reg.gauss_newton_step(corr, rk.RigidTransform.identity(), 1e9)
    r = reg.point_to_plane_residuals(corr, rk.RigidTransform.identity())
    J = np.concatenate([np.cross(p, n), n], axis=1)
    assert np.abs(xi - np.linalg.solve(J.T @ J, -J.T @ r)).max() < 1e-9
    flat = np.zeros((100, 3))
    flat[:, :2] = g.normal(scale=2.0, size=(100, 2))
    plane = reg.CorrespondenceSet(flat, flat, np.tile([0.0, 0.0, 1.0], (100, 1)))
    with pytest.raises(rk.DegenerateGeometry):
        reg.gauss_newton_step(plane, rk.RigidTransform.identity(), 0.5)


# ---------------------------------------------------------------- TSDF (K4, K5)

def test_activation_bitexact(rk, golden_tsdf):
    grid = rk.VoxelBlockGrid(voxel_size=0.1)
    keys = rk.activate_blocks(golden_tsdf["act_pts"], grid, 0.55)
    assert sorted(keys) == [tuple(k) for k in golden_tsdf["act_keys"].tolist()]
    assert set(grid.blocks) == keys


def _seq_grid(rk, sensors, g):
    intr = sensors["small"]
    grid = rk.VoxelBlockGrid(voxel_size=0.2)
    counts = []
    for f, M in zip(g["seq_frames"], g["seq_poses"]):
        counts.append(rk.integrate_cloud_frame(grid, rk.RangeImage(f, intr),
                                               rk.RigidTransform(M[:3, :3], M[:3, 3]), clip_max=12.0))
    return grid, counts


def _grid_vox(grid):
    items = sorted(grid.blocks.items())
    keys = [k for k, _ in items]
    vox = np.stack([np.stack([b.tsdf.reshape(-1), b.weight.reshape(-1)], -1) for _, b in items])
    return keys, vox


def test_tsdf_sequence_cr_bitexact_vs_oracle(rk, sensors, osensors, golden_tsdf):
    from oracle import tsdf as otsdf
    from paper_2112_02779_b200 import lidar_model as lm
    g = golden_tsdf
    with lm.math_mode(lm.MATH_CR):
        grid, counts = _seq_grid(rk, sensors, g)
    og, oc = {}, []
    for f, M in zip(g["seq_frames"], g["seq_poses"]):
        oc.append(otsdf.integrate_cloud_frame(og, osensors["small"], f, M[:3, :3], M[:3, 3], 0.2, 0.8,
                                              clip_max=12.0, math="cr")[1])
    assert counts == oc
    keys, vox = _grid_vox(grid)
    assert keys == sorted(og)
    ovox = np.stack([np.stack([og[k][0].reshape(-1), og[k][1].reshape(-1)], -1) for k in keys])
    assert np.array_equal(vox, ovox)


@pytest.mark.usefixtures("fast_math")
def test_tsdf_sequence_vs_reference(rk, sensors, golden_tsdf):
    g = golden_tsdf
    grid, counts = _seq_grid(rk, sensors, g)
    keys, vox = _grid_vox(grid)
    assert keys == [tuple(k) for k in g["seq_keys"].tolist()]            # bit-exact allocation
    ref = g["seq_vox"]
    assert np.mean(vox[..., 1] == ref[..., 1]) >= 0.9999
    same_w = vox[..., 1] == ref[..., 1]
    assert np.mean(np.abs(vox[..., 0] - ref[..., 0])[same_w] <= 1e-5) >= 0.9999
    assert np.all(np.abs(np.array(counts) - g["seq_counts"]) <= np.maximum(3, 1e-3 * g["seq_counts"]))
    s, w, ok = rk.query_sdf_many(grid, g["q_pts"])
    assert np.mean(ok == g["q_ok"]) >= 0.99


@pytest.mark.usefixtures("fast_math")
def test_tsdf_street_frame_vs_reference(rk, sensors, golden_tsdf, golden_icp):
    g = golden_tsdf
    grid = rk.VoxelBlockGrid(voxel_size=0.05)
    n = rk.integrate_cloud_frame(grid, rk.RangeImage(golden_icp["street/dst"], sensors["ouster"]),
                                 rk.RigidTransform.identity(), clip_max=30.0)
    keys = sorted(grid.blocks)
    assert keys == [tuple(k) for k in g["street_keys"].tolist()]
    assert abs(n - int(g["street_count"])) <= 1e-4 * int(g["street_count"]) + 5
    items = dict(grid.blocks.items())
    for j, i in enumerate(g["street_pick"]):
        b = items[keys[i]]
        ref = g["street_pick_vox"][j]
        assert np.mean(b.weight.reshape(-1) == ref[:, 1]) >= 0.999
        assert np.mean(np.abs(b.tsdf.reshape(-1) - ref[:, 0]) <= 1e-5) >= 0.999


def test_integrate_sequence_graph_replay_matches_eager(rk, sensors, golden_icp):
    """pipeline.integrate_sequence(graph=True): the recorded launches replayed
    on a cleared grid reproduce the eager sequence bit for bit (frame stamps
    and block counters live on the device)."""
    import torch
    from paper_2112_02779_b200 import pipeline, scenes
    intr = sensors["ouster"]
    traj = scenes.street_trajectory(6, seed=0)
    frames = pipeline.render_batch(intr, scenes.street_scene(), traj)
    poses = torch.from_numpy(pipeline.poses_to_rows(traj)).cuda()
    inv = torch.from_numpy(np.stack([p.inverse().as_row12() for p in traj])).cuda()
    out = []
    upd = torch.zeros(1, dtype=torch.int64, device="cuda")
    for graph in (False, True, True):
        grid = rk.VoxelBlockGrid(voxel_size=0.05, capacity=8192) if not out else out_grid
        pipeline.clear_grid(grid)
        upd.zero_()
        pipeline.integrate_sequence(grid, intr, frames, poses, inv, clip_max=30.0, updated=upd,
                                    graph=graph)
        keys, vox = _grid_vox(grid)
        out.append((int(upd.item()), keys, vox))
        out_grid = grid
    assert len(out_grid._graphs) == 1          # recorded once, replayed once
    for n, keys, vox in out[1:]:
        assert n == out[0][0] and keys == out[0][1] and np.array_equal(vox, out[0][2])


def test_integrate_sequence_graph_cache_owns_its_buffers(rk, sensors):
    """graph=True without caller-provided inverse poses / counter: the cache
    entry owns those buffers, so repeated calls replay ONE graph (the cache
    does not grow per call) and each call returns a fresh count equal to the
    eager run's; the cache is bounded by VoxelBlockGrid.MAX_GRAPHS."""
    import torch
    from paper_2112_02779_b200 import pipeline, scenes
    intr = sensors["ouster"]
    traj = scenes.street_trajectory(4, seed=1)
    frames = pipeline.render_batch(intr, scenes.street_scene(), traj)
    poses = torch.from_numpy(pipeline.poses_to_rows(traj)).cuda()
    grid = rk.VoxelBlockGrid(voxel_size=0.05, capacity=8192)
    ref = int(pipeline.integrate_sequence(grid, intr, frames, poses, clip_max=30.0).item())
    counts = []
    for _ in range(3):
        pipeline.clear_grid(grid)
        counts.append(pipeline.integrate_sequence(grid, intr, frames, poses, clip_max=30.0, graph=True))
    assert len(grid._graphs) == 1
    assert [int(c.item()) for c in counts] == [ref] * 3
    assert len({c.data_ptr() for c in counts}) == 3       # kept results are not overwritten
    for i in range(grid.MAX_GRAPHS + 3):
        grid.cache_graph(("probe", i), None)
    assert len(grid._graphs) == grid.MAX_GRAPHS


def test_sharded_grid_overflow_raises(rk, sensors):
    """ShardedGrid.integrate_frames with an undersized pool raises instead of
    silently skipping the unallocated blocks (eager and on the first replay
    of a recorded graph)."""
    import torch
    from paper_2112_02779_b200 import pipeline, scenes
    from paper_2112_02779_b200.distributed import ShardedGrid
    intr = sensors["ouster"]
    traj = scenes.street_trajectory(2, seed=0)
    frames = pipeline.render_batch(intr, scenes.street_scene(), traj)
    poses = torch.from_numpy(pipeline.poses_to_rows(traj)).cuda()
    inv = torch.from_numpy(np.stack([p.inverse().as_row12() for p in traj])).cuda()
    for graph in (False, True):
        sg = ShardedGrid(0.05, 0, 1, capacity=64)
        with pytest.raises(rk.DeviceError, match="overflow"):
            sg.integrate_frames(intr, frames, poses, inv, clip_max=30.0, graph=graph)


def test_hash_sharded_grid_equals_single_grid(rk, sensors, golden_icp):
    """Two block shards (emulated in one process) reproduce the unsharded grid
    bit for bit, including the global sorted-chunk arithmetic."""
    import torch
    from paper_2112_02779_b200 import _native as nat
    from paper_2112_02779_b200 import lidar_model as lm
    intr = sensors["ouster"]
    frame = torch.from_numpy(golden_icp["street/dst"]).cuda()
    pose = rk.RigidTransform.identity()
    full = rk.VoxelBlockGrid(voxel_size=0.05, capacity=8192)
    n_full = rk.integrate_cloud_frame(full, rk.RangeImage(frame, intr), pose, clip_max=30.0)
    shards = [rk.VoxelBlockGrid(voxel_size=0.05, capacity=8192) for _ in range(2)]
    st = nat.stream_ptr()
    p12 = nat.to_dev(pose.as_row12(), np.float64)
    inv = nat.to_dev(pose.inverse().as_row12(), np.float64)
    stats = [nat.zeros((2,), np.int64) for _ in range(2)]
    for r, g in enumerate(shards):
        h = g._ensure()
        nat.call("rk_grid_set_shard", h, r, 2)
        nat.call("rk_grid_activate_image", h, lm.device_sensor(intr), nat.ptr(frame), nat.ptr(p12),
                 float(g.truncation), 0.0, 30.0, st)
        nat.call("rk_grid_touch_stats", h, nat.ptr(stats[r]), st)
    glob = torch.stack([stats[0][0] + stats[1][0], torch.maximum(stats[0][1], stats[1][1])])
    upd = nat.zeros((1,), np.int64)
    for g in shards:
        nat.call("rk_grid_set_global_touch", g._handle, nat.ptr(glob))
        nat.call("rk_grid_integrate", g._handle, lm.device_sensor(intr), nat.ptr(frame), nat.ptr(inv),
                 0.0, 30.0, lm.default_math(), nat.ptr(upd), st)
        g.blocks._bump()
    assert int(upd.item()) == n_full
    k0, k1 = set(shards[0].blocks), set(shards[1].blocks)
    assert not (k0 & k1) and (k0 | k1) == set(full.blocks)
    fb = dict(full.blocks.items())
    for g in shards:
        for k, b in g.blocks.items():
            assert np.array_equal(b.tsdf, fb[k].tsdf) and np.array_equal(b.weight, fb[k].weight)


def test_sharded_batched_sequence_equals_single_grid(rk, sensors):
    """The multi-GPU TSDF flow (ShardedGrid.integrate_frames: F activations
    into F slots, one reduction of the per-frame {count, max key}, F
    integrations), emulated with two shards in one process, reproduces the
    unsharded sequence bit for bit."""
    import torch
    from paper_2112_02779_b200 import _native as nat
    from paper_2112_02779_b200 import lidar_model as lm
    from paper_2112_02779_b200 import pipeline, scenes
    intr = sensors["ouster"]
    traj = scenes.street_trajectory(5, seed=0)
    frames = pipeline.render_batch(intr, scenes.street_scene(), traj)
    poses = torch.from_numpy(pipeline.poses_to_rows(traj)).cuda()
    inv = torch.from_numpy(np.stack([p.inverse().as_row12() for p in traj])).cuda()
    full = rk.VoxelBlockGrid(voxel_size=0.05, capacity=8192)
    n_full = pipeline.integrate_sequence(full, intr, frames, poses, inv, clip_max=30.0)
    F, st = frames.shape[0], nat.stream_ptr()
    sensor = lm.device_sensor(intr)
    shards = [rk.VoxelBlockGrid(voxel_size=0.05, capacity=8192) for _ in range(2)]
    stats = []
    for r, g in enumerate(shards):
        h = g._ensure()
        nat.call("rk_grid_set_shard", h, r, 2)
        nat.call("rk_grid_reserve_slots", h, F, st)
        nat.call("rk_grid_activate_frames", h, sensor, nat.ptr(frames), F, nat.ptr(poses),
                 float(g.truncation), 0.0, 30.0, st)
        s2 = nat.zeros((F, 2), np.int64)
        nat.call("rk_grid_touch_stats_frames", h, F, nat.ptr(s2), st)
        stats.append(s2)
    glob = torch.stack([stats[0][:, 0] + stats[1][:, 0], torch.maximum(stats[0][:, 1], stats[1][:, 1])],
                       -1).contiguous()
    upd = nat.zeros((1,), np.int64)
    for g in shards:
        nat.call("rk_grid_integrate_activated", g._handle, sensor, nat.ptr(frames), F, nat.ptr(inv),
                 nat.ptr(glob), 0.0, 30.0, lm.default_math(), nat.ptr(upd), st)
        g.blocks._bump()
    assert int(upd.item()) == int(n_full.item())
    kf, vf = full.export_blocks()
    parts = [g.export_blocks() for g in shards]
    k = np.concatenate([p[0] for p in parts])
    v = np.concatenate([p[1] for p in parts])
    order = np.lexsort((k[:, 2], k[:, 1], k[:, 0]))
    assert np.array_equal(k[order], kf) and np.array_equal(v[order], vf)


def test_sharded_mesh_with_halo_equals_single_grid(rk, sensors):
    """Distributed marching cubes (two shards emulated in one process): each
    shard meshes its own blocks with the other's boundary blocks as halo; the
    merged mesh equals the single-grid mesh (same vertex positions, same
    triangles up to relabelling)."""
    import torch
    from paper_2112_02779_b200 import _native as nat
    from paper_2112_02779_b200 import distributed as rkd
    from paper_2112_02779_b200 import pipeline, scenes
    intr = sensors["ouster"]
    traj = scenes.street_trajectory(3, seed=0)
    frames = pipeline.render_batch(intr, scenes.street_scene(), traj)
    poses = torch.from_numpy(pipeline.poses_to_rows(traj)).cuda()
    inv = torch.from_numpy(np.stack([p.inverse().as_row12() for p in traj])).cuda()
    full = rk.VoxelBlockGrid(voxel_size=0.1, capacity=4096)
    pipeline.integrate_sequence(full, intr, frames, poses, inv, clip_max=30.0)
    ref = rk.extract_mesh(full)
    keys, vox = full.export_blocks(device=True)
    owner = torch.from_numpy(rkd.block_owner(nat.to_host(keys), 2)).cuda()
    shards = []
    for r in range(2):
        g = rk.VoxelBlockGrid(voxel_size=0.1, capacity=4096)
        m = owner == r
        g.import_blocks(keys[m], vox[m])
        shards.append(g)
    by_rank = [s.export_blocks(device=True) for s in shards]
    plan = rkd.halo_plan([nat.to_host(k) for k, _ in by_rank])
    parts = []
    for r in range(2):
        o = 1 - r
        sel = torch.from_numpy(plan[o][r]).cuda()
        parts.append(rkd.mesh_from_shard(shards[r], r, 2, by_rank[o][0][sel], by_rank[o][1][sel]))
    V, T, N = rkd.merge_meshes(parts)
    assert V.shape[0] == ref.n_vertices and T.shape[0] == ref.n_triangles > 1000
    pos = {tuple(p): i for i, p in enumerate(ref.vertices.tolist())}
    remap = np.array([pos[tuple(p)] for p in V.tolist()])
    assert np.abs(N - ref.normals[remap]).max() < 1e-12
    canon = lambda tris: {tuple(np.roll(t, -int(np.argmin(t)))) for t in tris.tolist()}  # noqa: E731
    assert canon(remap[T]) == canon(ref.triangles)


def test_integrate_rejects_bad_pose(rk, sensors, golden_icp):
    grid = rk.VoxelBlockGrid(voxel_size=0.1)
    img = rk.RangeImage(golden_icp["synth/dst"], sensors["synth"])
    with pytest.raises(rk.InvalidPose):
        rk.integrate(grid, img, rk.RigidTransform(np.eye(3) * 2.0, np.zeros(3)), set())


def test_block_mapping_roundtrip(rk):
    grid = rk.VoxelBlockGrid(voxel_size=0.1)
    blk = rk.VoxelBlock()
    blk.tsdf = np.arange(4096, dtype=np.float32).reshape(16, 16, 16) / 4096
    blk.weight = np.ones((16, 16, 16), np.float32)
    grid.blocks[(1, -2, 3)] = blk
    assert (1, -2, 3) in grid.blocks and len(grid.blocks) == 1
    grid.reserve(4096)  # forces a flush + rehash
    got = grid.blocks[(1, -2, 3)]
    assert np.array_equal(got.tsdf, blk.tsdf) and np.array_equal(got.weight, blk.weight)


# ---------------------------------------------------------------- marching cubes (K6)

def _mesh_grid(rk, g):
    grid = rk.VoxelBlockGrid(voxel_size=0.05, truncation=0.2)
    for k, v in zip(g["sphere_keys"].tolist(), g["sphere_vox"]):
        grid.blocks[tuple(k)] = rk.VoxelBlock(v[:, 0].reshape(16, 16, 16).copy(),
                                              v[:, 1].reshape(16, 16, 16).copy())
    return grid


def test_mesh_sphere_vs_reference(rk, golden_mesh):
    g = golden_mesh
    m = rk.extract_mesh(_mesh_grid(rk, g))
    V, T, N = g["sphere_V"], g["sphere_T"], g["sphere_N"]
    assert m.n_vertices == V.shape[0] and m.n_triangles == T.shape[0]
    pos = {tuple(p): i for i, p in enumerate(V.tolist())}
    remap = np.array([pos[tuple(p)] for p in m.vertices.tolist()])       # exact positions
    assert len(set(remap.tolist())) == V.shape[0]
    assert np.abs(m.normals - N[remap]).max() < 1e-12
    canon = lambda tris: {tuple(np.roll(t, -int(np.argmin(t)))) for t in tris.tolist()}  # noqa: E731
    assert canon(remap[m.triangles]) == canon(T)


def test_mesh_empty_and_uniform(rk):
    grid = rk.VoxelBlockGrid(voxel_size=0.05)
    m = rk.extract_mesh(grid)
    assert m.n_vertices == 0 and m.n_triangles == 0
    blk = rk.VoxelBlock(np.full((16, 16, 16), 0.2, np.float32), np.ones((16, 16, 16), np.float32))
    grid.blocks[(0, 0, 0)] = blk
    m = rk.extract_mesh(grid)
    assert m.n_vertices == 0 and m.n_triangles == 0


def test_smoke_entry():
    import __graft_entry__
    __graft_entry__.smoke()


# ---------------------------------------------------------------- SURVEY §8(f) rows

@pytest.mark.parametrize("pair", ("room", "street"))
def test_from_point_cloud_vs_reference(rk, pair, sensors, golden_next):
    """N1: float64 projection + atomicMin z-buffer against the reference's
    from_point_cloud (device float64 atan2/sin/cos may differ from numpy's in
    the last ulp, so a pixel may rarely change hands)."""
    g = golden_next
    img, st = rk.from_point_cloud(g[f"{pair}/fpc_in"], sensors[SENSOR_OF[pair]])
    ref = g[f"{pair}/fpc_img"]
    assert img.data.dtype == np.float32 and img.data.shape == ref.shape
    assert np.mean(img.data == ref) >= 0.9999
    assert np.abs(img.data - ref).max() <= 1e-4 or np.mean(img.data != ref) < 1e-4
    k = g[f"{pair}/fpc_stats"]
    assert (st.out_of_fov, st.degenerate) == (int(k[2]), int(k[3]))
    assert abs(st.kept - int(k[0])) <= 2 and abs(st.collisions - int(k[1])) <= 2
    assert st.kept + st.collisions == int(k[0] + k[1])


def test_from_point_cloud_device_and_empty(rk, sensors):
    import torch
    intr = sensors["small"]
    img, st = rk.from_point_cloud(np.zeros((0, 3)), intr)
    assert not img.data.any() and (st.kept, st.collisions, st.out_of_fov, st.degenerate) == (0, 0, 0, 0)
    pts = torch.tensor([[5.0, 0.0, 0.0], [5.0, 0.001, 0.0], [6.0, 0.0, 0.0]], device="cuda",
                       dtype=torch.float64)
    img, st = rk.from_point_cloud(pts, intr)
    assert img.on_device
    assert st.kept + st.collisions == 3 and st.kept >= 1
    assert float(img.data[img.data > 0].min()) < 5.1      # nearest range wins


@pytest.mark.parametrize("pair", ("room", "synth"))
def test_pca_normals_vs_reference(rk, pair, sensors, golden_icp, golden_next):
    """N3: valid masks exactly (window counts are exact arithmetic), normals
    within 1e-5 of numpy's eigh wherever the smallest eigenvalue is separated."""
    g = golden_next
    img = rk.RangeImage(golden_icp[f"{pair}/dst"], sensors[SENSOR_OF[pair]])
    for key, kw in (("pca", {}), ("pca1", dict(radius=1, discontinuity_abs=0.1,
                                                discontinuity_rel=0.02))):
        nm = rk.compute_normal_map(img, "pca", **kw)
        assert np.array_equal(nm.valid, g[f"{pair}/{key}_valid"])
        d = np.abs(nm.vectors - g[f"{pair}/{key}_nrm"]).max(axis=-1)[nm.valid]
        assert np.mean(d <= 1e-5) >= 0.999, (key, np.mean(d <= 1e-5))


@pytest.mark.parametrize("pair", ("room", "synth"))
def test_register_pca_normals_vs_reference(rk, pair, sensors, golden_icp, golden_next):
    g = golden_next
    intr = sensors[SENSOR_OF[pair]]
    res = rk.register(rk.RangeImage(golden_icp[f"{pair}/src"], intr),
                      rk.RangeImage(golden_icp[f"{pair}/dst"], intr),
                      config=rk.RegistrationConfig(normal_method="pca"))
    M = g[f"{pair}/pca_reg_pose"]
    assert rot_err(res.pose.R, M[:3, :3]) < 1e-5 and np.linalg.norm(res.pose.t - M[:3, 3]) < 1e-5
    got = np.array([[s.stride, s.iteration] for s in res.stats])
    assert np.array_equal(got, g[f"{pair}/pca_reg_stats"][:, :2])


def test_sdfg_round_trip_bytes_and_values(rk, sensors, golden_tsdf, golden_next, tmp_path):
    """N2: the reference's SDFG snapshot loads into the device grid and writes
    back byte for byte; a grid integrated on the device exports the same key
    set with values within the TSDF tolerance."""
    from paper_2112_02779_b200 import io_formats
    blob = golden_next["sdfg_bytes"].tobytes()
    (tmp_path / "ref.sdfg").write_bytes(blob)
    grid = io_formats.read_grid(tmp_path / "ref.sdfg")
    io_formats.write_grid(tmp_path / "back.sdfg", grid)
    assert (tmp_path / "back.sdfg").read_bytes() == blob
    mine, _ = _seq_grid(rk, sensors, golden_tsdf)
    io_formats.write_grid(tmp_path / "mine.sdfg", mine)
    a = io_formats.read_grid(tmp_path / "mine.sdfg").export_blocks()
    b = grid.export_blocks()
    assert np.array_equal(a[0], b[0])
    same_w = a[1][..., 1] == b[1][..., 1]
    assert np.mean(same_w) >= 0.9999
    assert np.mean(np.abs(a[1][..., 0] - b[1][..., 0])[same_w] <= 1e-5) >= 0.9999
    with pytest.raises(rk.FormatError):
        (tmp_path / "bad.sdfg").write_bytes(b"XXXX" + blob[4:])
        io_formats.read_grid(tmp_path / "bad.sdfg")
    with pytest.raises(rk.TruncatedPayload):
        (tmp_path / "short.sdfg").write_bytes(blob[:100])
        io_formats.read_grid(tmp_path / "short.sdfg")


def test_register_single_plane_is_degenerate(rk, sensors, osensors):
    """A single plane leaves three DoF unobservable: the reference raises
    DegenerateGeometry (cond(H) > 1e12, registration.py:270-272); the
    warp-parallel update must route it to the exact test and agree."""
    import torch
    from oracle import synth as osynth
    intr = sensors["small"]
    img = osynth.render(osensors["small"], [("plane", (1.0, 0.0, 0.0), -4.0)])
    assert (img > 0).sum() > 1000
    with pytest.raises(rk.DegenerateGeometry):
        rk.register(rk.RangeImage(img, intr), rk.RangeImage(img, intr))
    t = torch.from_numpy(img).cuda()[None].repeat(2, 1, 1)
    res = rk.register_batch(intr, t, t)
    assert res.status.tolist() == [2, 2]


def test_nvtx_tracing_is_transparent(rk, sensors, golden_icp):
    """RK_NVTX-style tracing wraps the public calls without changing results."""
    from paper_2112_02779_b200 import trace
    intr = sensors["synth"]
    src, dst = rk.RangeImage(golden_icp["synth/src"], intr), rk.RangeImage(golden_icp["synth/dst"], intr)
    a = rk.register(src, dst)
    trace.enable(True)
    try:
        b = rk.register(src, dst)
    finally:
        trace.enable(False)
    assert np.array_equal(a.pose.matrix(), b.pose.matrix())


def test_grid_pool_growth_is_transparent(rk, sensors, golden_tsdf, golden_icp):
    """A pool far too small for the data (capacity 4 blocks) grows on
    overflow and re-runs the activation: the per-call API leaves exactly the
    grid and counts of a pre-sized pool (activate_blocks and
    integrate_cloud_frame, sdf_volume.py:82-113, 198-210).  The batched
    sequence path reports the overflow instead (caller-sized pool)."""
    import torch
    from paper_2112_02779_b200 import pipeline
    small = rk.VoxelBlockGrid(voxel_size=0.1, capacity=4)
    keys = rk.activate_blocks(golden_tsdf["act_pts"], small, 0.55)
    assert sorted(keys) == [tuple(k) for k in golden_tsdf["act_keys"].tolist()]
    assert small.info()[1] > 4 and not small.info()[2]
    intr = sensors["ouster"]
    frame = golden_icp["street/dst"]
    pose = rk.RigidTransform.identity()
    a = rk.VoxelBlockGrid(voxel_size=0.05, capacity=4)
    b = rk.VoxelBlockGrid(voxel_size=0.05, capacity=16384)
    for _ in range(2):
        na = rk.integrate_cloud_frame(a, rk.RangeImage(frame, intr), pose, clip_max=30.0)
        nb = rk.integrate_cloud_frame(b, rk.RangeImage(frame, intr), pose, clip_max=30.0)
        assert na == nb
    ka, va = a.export_blocks()
    kb, vb = b.export_blocks()
    assert np.array_equal(ka, kb) and np.array_equal(va, vb)
    c = rk.VoxelBlockGrid(voxel_size=0.05, capacity=4)
    dev = torch.from_numpy(frame).cuda()[None]
    rows = torch.from_numpy(pipeline.poses_to_rows([pose])).cuda()
    pipeline.integrate_sequence(c, intr, dev, rows)
    assert c.info()[2] == 1            # overflow flagged, never silent


def test_register_batch_bad_pair_index(rk, sensors, golden_icp):
    """Pair indices outside the image pools are caught on the device: the
    pair gets ICP_BAD_PAIR and its init pose, no out-of-bounds read, and the
    other pairs of the batch are unaffected."""
    import torch
    from paper_2112_02779_b200.registration import ICP_BAD_PAIR
    intr = sensors["ouster"]
    src = torch.from_numpy(golden_icp["street/src"]).cuda()[None].repeat(2, 1, 1)
    dst = torch.from_numpy(golden_icp["street/dst"]).cuda()[None].repeat(2, 1, 1)
    ok = rk.register_batch(intr, src, dst)
    ps = torch.tensor([0, 5, 1, -1], dtype=torch.int32, device="cuda")
    pd = torch.tensor([0, 1, 7, 1], dtype=torch.int32, device="cuda")
    res = rk.register_batch(intr, src, dst, pair_src=ps, pair_dst=pd)
    st = res.status.cpu().numpy()
    assert list(st[1:]) == [ICP_BAD_PAIR] * 3 and st[0] == int(ok.status[0].item())
    assert torch.equal(res.poses[0], ok.poses[0])
    eye = torch.tensor([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], dtype=torch.float64, device="cuda")
    assert all(torch.equal(res.poses[i], eye) for i in (1, 2, 3))
    assert res.iterations[1:].abs().sum().item() == 0


def test_sharded_frames_graph_replay_matches_eager(rk, sensors):
    """ShardedGrid.integrate_frames(graph=True): the two recorded phases
    (activation of all F frames + stats export; the F integrations) replayed
    around the collective reproduce the eager flow bit for bit, for a lone
    grid and for each of two emulated shards (the collective replaced by the
    precomputed global {count, max key} pairs)."""
    import torch
    from paper_2112_02779_b200 import distributed as rkd
    from paper_2112_02779_b200 import pipeline, scenes
    intr = sensors["ouster"]
    traj = scenes.street_trajectory(5, seed=0)
    frames = pipeline.render_batch(intr, scenes.street_scene(), traj)
    poses = torch.from_numpy(pipeline.poses_to_rows(traj)).cuda()
    inv = torch.from_numpy(np.stack([p.inverse().as_row12() for p in traj])).cuda()
    # lone grid (world 1): eager vs record + replay
    lone = rkd.ShardedGrid(0.05, 0, 1, capacity=8192)
    ref = None
    for graph in (False, True, True):
        pipeline.clear_grid(lone.grid)
        upd = torch.zeros(1, dtype=torch.int64, device="cuda")
        lone.integrate_frames(intr, frames, poses, inv, clip_max=30.0, updated=upd, graph=graph)
        k, v = lone.grid.export_blocks()
        if ref is None:
            ref = (int(upd.item()), k, v)
        else:
            assert int(upd.item()) == ref[0] and np.array_equal(k, ref[1]) and np.array_equal(v, ref[2])
    # two shards: global stats from an eager activation pass of both
    shards = [rkd.ShardedGrid(0.05, r, 2, capacity=8192) for r in range(2)]
    stats = []
    for sh in shards:
        sh.integrate_frames(intr, frames, poses, inv, clip_max=30.0,
                            reduce=lambda st: stats.append(st.clone()) or st)
    glob = torch.stack([stats[0][:, 0] + stats[1][:, 0], torch.maximum(stats[0][:, 1], stats[1][:, 1])],
                       -1).contiguous()
    for sh in shards:
        outs = []
        for graph in (False, True, True):
            pipeline.clear_grid(sh.grid)
            upd = torch.zeros(1, dtype=torch.int64, device="cuda")
            sh.integrate_frames(intr, frames, poses, inv, clip_max=30.0, updated=upd, graph=graph,
                                reduce=lambda st: glob)
            outs.append((int(upd.item()),) + sh.grid.export_blocks())
        for n, k, v in outs[1:]:
            assert n == outs[0][0] and np.array_equal(k, outs[0][1]) and np.array_equal(v, outs[0][2])
    # and the shards together equal the lone grid
    k = np.concatenate([sh.grid.export_blocks()[0] for sh in shards])
    assert len(k) == len(ref[1])


@pytest.mark.timeout(300)
def test_register_ill_conditioned_corridor_terminates(rk):
    """Regression: a pair whose normal equations fall in the band between the
    condition-number bounds (the sensor drifted below the ground slab of the
    C5 extended street: a corridor of parallel planes) takes the exact serial
    fallback; the warp-parallel update once let lanes 0-7 branch into it while
    lanes 8-31 continued (a non-uniform trace bound), deadlocking the warp's
    full-mask shuffles.  It must finish with a defined status."""
    import torch
    from paper_2112_02779_b200 import pipeline, scenes
    from paper_2112_02779_b200.registration import ICP_BAD_PAIR
    intr = scenes.os128()
    traj = scenes.street_trajectory(438, seed=0, step_m=0.5)   # default 2 mrad jitter
    frames = pipeline.render_batch(intr, scenes.extended_street_scene(330.0), traj[436:438])
    res = rk.register_batch(intr, frames[1:2], frames[0:1])
    torch.cuda.synchronize()
    st = int(res.status[0].item())
    assert st in (0, 1, 2) and st != ICP_BAD_PAIR
    assert torch.isfinite(res.poses).all()


@pytest.mark.timeout(300)
def test_register_batch_stress_terminates(rk):
    """Termination and defined outputs on hostile inputs, one batch: large
    perturbations (up to 25 deg / 4 m), 5-cm range noise, all-sky and empty
    images, a sensor below the ground, and the C5 corridor pairs whose
    normal equations are singular or in the condition bounds' band."""
    import torch
    from paper_2112_02779_b200 import pipeline, scenes
    intr = scenes.ouster64()
    street = scenes.street_scene()
    g = np.random.default_rng(123)
    dst_poses, src_poses = [], []
    for k in range(96):
        yaw = g.uniform(-np.pi, np.pi)
        base = rk.RigidTransform.exp(np.array([0, 0, yaw, g.uniform(-4, 4), g.uniform(-9, 9),
                                               g.uniform(-3.0, 0.5)]))
        pert = scenes.perturbation_pose(np.random.default_rng(k), g.uniform(0, 25), g.uniform(0, 4))
        dst_poses.append(base)
        src_poses.append(base @ pert)
    dst = pipeline.render_batch(intr, street, dst_poses)
    src = pipeline.render_batch(intr, street, src_poses)
    noise = torch.randn_like(src) * 0.05
    src = torch.where(src > 0, (src + noise).clamp_min(0.0), src)
    src[0] = 0.0                      # empty source
    dst[1] = 0.0                      # empty destination
    src[2, 20:] = 0.0                 # mostly sky
    res = rk.register_batch(intr, src, dst)
    torch.cuda.synchronize()
    st = res.status.cpu().numpy()
    assert set(np.unique(st)) <= {0, 1, 2}
    assert torch.isfinite(res.poses).all()
    assert st[0] == 1 and st[1] == 1
    # the C5 corridor: a jittered 500-frame drive that leaves the street
    c5 = scenes.os128()
    traj = scenes.street_trajectory(600, seed=0, step_m=0.5)
    frames = pipeline.render_batch(c5, scenes.extended_street_scene(330.0), traj[400:600])
    ps = torch.arange(1, 200, dtype=torch.int32, device="cuda")
    res = rk.register_batch(c5, frames, frames, pair_src=ps, pair_dst=ps - 1)
    torch.cuda.synchronize()
    st = res.status.cpu().numpy()
    assert set(np.unique(st)) <= {0, 1, 2} and (st == 2).any()
    assert torch.isfinite(res.poses).all()


def test_register_batch_validates_inputs(rk, sensors):
    """Shapes, dtypes and devices are checked on the host before any launch
    (a mis-shaped pool would otherwise be read out of bounds)."""
    import torch
    intr = sensors["ouster"]
    H, W = intr.height, intr.width
    good = torch.zeros((2, H, W), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        rk.register_batch(intr, torch.zeros((2, W, H), device="cuda"), good)
    with pytest.raises(ValueError):
        rk.register_batch(intr, good, good.double())
    with pytest.raises(ValueError):
        rk.register_batch(intr, good.cpu(), good)
    with pytest.raises(ValueError):
        rk.register_batch(intr, good, good, torch.zeros((2, H, W, 3), device="cuda"))
    with pytest.raises(ValueError):
        rk.register_batch(intr, good, good, pair_src=torch.zeros(2, dtype=torch.int32, device="cuda"))


def test_register_host_graph_path_equals_device_path(rk, sensors, golden_icp):
    """register() on host images replays one recorded CUDA graph (H2D, K1,
    K3, D2H); its results equal the eager device-image path bit for bit,
    also on a second call with other images (the staging buffers refill)."""
    import torch
    g, intr = golden_icp, sensors["ouster"]
    for src, dst in ((g["street/src"], g["street/dst"]), (g["street/dst"], g["street/src"])):
        a = rk.register(rk.RangeImage(src, intr), rk.RangeImage(dst, intr))
        b = rk.register(rk.RangeImage(torch.from_numpy(src).cuda(), intr),
                        rk.RangeImage(torch.from_numpy(dst).cuda(), intr))
        assert np.array_equal(a.pose.matrix(), b.pose.matrix())
        assert [(s.stride, s.iteration, s.n_correspondences, s.cost) for s in a.stats] == \
               [(s.stride, s.iteration, s.n_correspondences, s.cost) for s in b.stats]
        assert a.converged == b.converged
    init = rk.RigidTransform.exp(np.array([0.01, 0.0, 0.02, 0.1, -0.05, 0.0]))
    a = rk.register(rk.RangeImage(g["street/src"], intr), rk.RangeImage(g["street/dst"], intr), init=init)
    b = rk.register(rk.RangeImage(torch.from_numpy(g["street/src"]).cuda(), intr),
                    rk.RangeImage(torch.from_numpy(g["street/dst"]).cuda(), intr), init=init)
    assert np.array_equal(a.pose.matrix(), b.pose.matrix())
