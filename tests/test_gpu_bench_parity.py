"""Parity on the benchmark's own workload: a random subset
of the device-rendered pool of street pairs is registered in one batched
launch and by the CPU oracle on the same images.

Pairs the reference algorithm solves (the oracle recovers the ground truth)
must agree within the north star's 1e-5 rad / 1e-5 m with identical
iteration counts.  A few pool pairs are ill-posed for point-to-plane ICP
(the oracle itself ends metres from the ground truth after all 50
iterations); their trajectories amplify any last-bit difference -- even the
exact MATH_CR mode, which differs from the oracle only in float32
summation order, ends 1e-3..1e-2 away -- so for them the contract is the
same outcome class: not recovered by either side."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_c4_pool_subset_vs_oracle():
    import torch

    import paper_2112_02779_b200 as rk
    from oracle import icp as oicp
    from oracle import image as oimg
    from oracle import sensor as osens
    from paper_2112_02779_b200 import pipeline, scenes
    intr = scenes.ouster64()
    S = osens.Sensor.from_intrinsics(intr)
    street = scenes.street_scene()
    pool = scenes.pair_pool_poses(2048, seed=0)
    pick = np.random.default_rng(2026).choice(len(pool), size=48, replace=False)
    dst_poses = [pool[i][0] for i in pick]
    src_poses = [pool[i][0] @ pool[i][1] for i in pick]
    src = pipeline.render_batch(intr, street, src_poses)
    dst = pipeline.render_batch(intr, street, dst_poses)
    res = rk.register_batch(intr, src, dst, with_stats=True)
    poses = res.poses.cpu().numpy()
    iters = res.iterations.cpu().numpy()
    src_h, dst_h = src.cpu().numpy(), dst.cpu().numpy()
    agree = well = 0
    gt = np.stack([pool[i][1].as_row12() for i in pick])
    for b in range(len(pick)):
        vec, valid = oimg.normals_cross(S, dst_h[b])
        ref = oicp.register(S, src_h[b], dst_h[b], vec, valid, math="cr", fma="exact")
        R, t = poses[b, :9].reshape(3, 3), poses[b, 9:]
        ref_ok = np.linalg.norm(ref["t"] - gt[b, 9:]) < 0.05
        gpu_ok = np.linalg.norm(t - gt[b, 9:]) < 0.05
        assert ref_ok == gpu_ok, b
        if ref_ok:
            well += 1
            agree += (np.abs(R - ref["R"]).max() < 1e-5 and np.abs(t - ref["t"]).max() < 1e-5
                      and int(iters[b]) == len(ref["stats"]))
    assert well >= 0.8 * len(pick)
    assert agree == well, f"{agree}/{well} well-posed pairs within tolerance"
