"""Parity on the benchmark's own workload against the
REFERENCE's own outputs: 256 pairs of the device-rendered pool, registered
by the unmodified reference (tests/golden/make_golden_c4.py, c4_pool.npz)
with one shard (threads=1) and with 2, 4 and 8 shards (8 = its default on
an 8-core host).

The bar is the reference's own reproducibility.  Its shard counts differ
only in how the float32 normal-equation sums of the stride-1 level are
split; across them every pair it solves ("well-posed": ends within 5 cm of
the ground truth) agrees within 1e-7 with identical iteration counts.  The
coarse levels are never split, so the golden file also holds the
reference with its float32 sums evaluated in float64 (``f64sum``: the same
per-point float32 terms, exact summation -- make_golden_c4.py).  The
reference's float32 sgemm is ~1e-5 relative from exact at the coarse
levels, and that alone moves one well-posed pair (pool pair 3: a
borderline level-exit test at stride 2 -> 39 instead of 50 iterations,
6e-5 away).  On the ill-posed pairs (ends metres away after all 50
iterations; the point-to-plane problem is nearly singular) the reference's
own runs disagree by up to 1e-4 -- chaotic, so only the outcome class is
compared.

The GPU, in the default MATH_NP mode, makes every projection decision
exactly as numpy does, computes every per-point float32 term exactly as
the reference does, and sums in a different (more accurate) order, so it is
held to: every well-posed pair within 1e-5, with the same iteration count,
of one of the reference's own results (threads=1 or f64sum), and no more
pairs away from threads=1 than f64sum itself is; every pair the same
outcome class.  MATH_FAST (opt-in) is reported with its own, wider bar.
"""

import hashlib
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden" / "c4_pool.npz"


@pytest.fixture(scope="module")
def c4():
    """The pool pairs rendered on the device (checked against the reference's
    render_scene bytes) and the reference's registration outputs."""
    import paper_2112_02779_b200 as rk
    from paper_2112_02779_b200 import pipeline, scenes
    g = dict(np.load(GOLDEN))
    intr = scenes.ouster64()
    pool = scenes.pair_pool_poses(2048, seed=0)
    pick = g["pick"]
    dst = pipeline.render_batch(intr, scenes.street_scene(), [pool[int(i)][0] for i in pick])
    src = pipeline.render_batch(intr, scenes.street_scene(), [pool[int(i)][0] @ pool[int(i)][1] for i in pick])
    sh, dh = src.cpu().numpy(), dst.cpu().numpy()
    bad = [b for b in range(len(pick)) if hashlib.sha1(sh[b].tobytes()).hexdigest() != str(g["src_sha1"][b])
           or hashlib.sha1(dh[b].tobytes()).hexdigest() != str(g["dst_sha1"][b])]
    assert not bad, f"device renderer differs from render_scene on pairs {bad[:8]}"
    gt = g["gt"]
    ref = g["t1/poses"]
    well = np.linalg.norm(ref[:, 9:] - gt[:, 9:], axis=1) < 0.05
    return dict(rk=rk, intr=intr, src=src, dst=dst, g=g, well=well)


def _reference_self_disagreement(g, well):
    """Pairs on which the reference's own threads=2/4/8 runs leave 1e-5 of its
    threads=1 run, or change the iteration count."""
    p1, it1 = g["t1/poses"], g["t1/iters"]
    out = {}
    for t in (2, 4, 8):
        d = np.nanmax(np.abs(g[f"t{t}/poses"] - p1), axis=1)
        flip = (d > 1e-5) | (g[f"t{t}/iters"] != it1)
        out[t] = (int(flip[well].sum()), int(flip[~well].sum()), float(np.nanmax(d[well])))
    return out


def _gpu(c4, mode):
    from paper_2112_02779_b200 import lidar_model as lm
    with lm.math_mode(mode):
        res = c4["rk"].register_batch(c4["intr"], c4["src"], c4["dst"], with_stats=True)
    return (res.poses.cpu().numpy(), res.iterations.cpu().numpy(), res.status.cpu().numpy(),
            res.stats.cpu().numpy())


def _flips(g, key, well):
    d = np.nanmax(np.abs(g[f"{key}/poses"] - g["t1/poses"]), axis=1)
    return (d > 1e-5) | (g[f"{key}/iters"] != g["t1/iters"])


def test_c4_reference_is_self_consistent_on_well_posed_pairs(c4):
    """The golden file's own properties the GPU bar rests on: the shard
    counts agree on every well-posed pair; exact summation moves at most a
    few of them."""
    g, well = c4["g"], c4["well"]
    assert well.sum() >= 0.85 * well.size
    for t, (nw, nill, dmax) in _reference_self_disagreement(g, well).items():
        assert nw == 0 and dmax < 1e-6, (t, nw, dmax)
    assert _flips(g, "f64sum", well)[well].sum() <= 3


def test_c4_np_vs_reference_threads1(c4):
    """MATH_NP (default): every well-posed pair within 1e-5 of one of the
    reference's own results with the same iteration count; on the threads=1
    trajectory the per-iteration correspondence counts equal the reference's
    (to the point on >= 99.5 % of iterations, within 2 points on all); every
    pair the same outcome class."""
    from paper_2112_02779_b200 import lidar_model as lm
    g, well = c4["g"], c4["well"]
    P, it, st, stats = _gpu(c4, lm.MATH_NP)
    ref, it1, gt = g["t1/poses"], g["t1/iters"], g["gt"]
    ok_gpu = np.linalg.norm(P[:, 9:] - gt[:, 9:], axis=1) < 0.05
    assert np.array_equal(ok_gpu, well)
    near_t1 = (np.abs(P - ref).max(axis=1) < 1e-5) & (it == it1)
    near_f64 = (np.nan_to_num(np.abs(P - g["f64sum/poses"]).max(axis=1), nan=1.0) < 1e-5) & \
        (it == g["f64sum/iters"])
    bad = np.nonzero(well & ~(near_t1 | near_f64))[0]
    assert bad.size == 0, bad
    assert (well & ~near_t1).sum() <= _flips(g, "f64sum", well)[well].sum()
    # per-iteration correspondence counts of the pairs on the threads=1 trajectory
    lens = g["t1/ncorr_len"]
    off = np.concatenate([[0], np.cumsum(lens)])
    same = total = absdiff = corr = 0
    for b in np.nonzero(well & near_t1)[0]:
        mine = stats[b, :it[b], 2].astype(np.int64)
        theirs = g["t1/ncorr_flat"][off[b]:off[b + 1]]
        assert np.all(np.abs(mine - theirs) <= 2), b
        same += int((mine == theirs).sum())
        total += len(theirs)
        absdiff += int(np.abs(mine - theirs).sum())
        corr += int(theirs.sum())
    # the poses differ by ~1e-8 (summation order): a point lying within that
    # of a decision boundary flips now and then -- a handful of points in
    # 3e8 correspondences, far inside the 99.9 % mask contract
    assert absdiff <= 1e-6 * corr, (absdiff, corr)
    assert same >= 0.995 * total, (same, total)


def test_c4_fast_vs_reference_threads1(c4):
    """MATH_FAST (opt-in: minimax transcendentals, MUFU square roots, float32
    move): the same outcome class on every pair; the well-posed pairs within
    the algorithm's own 1e-4 convergence tolerance, >= 97 % of them within
    1e-5 with the same iteration count (a borderline level-exit test moves
    by an iteration on a few pairs)."""
    from paper_2112_02779_b200 import lidar_model as lm
    g, well = c4["g"], c4["well"]
    P, it, st, _ = _gpu(c4, lm.MATH_FAST)
    ref, it1, gt = g["t1/poses"], g["t1/iters"], g["gt"]
    ok_gpu = np.linalg.norm(P[:, 9:] - gt[:, 9:], axis=1) < 0.05
    assert np.array_equal(ok_gpu, well)
    dev = np.abs(P - ref).max(axis=1)
    agree = (dev < 1e-5) & (it == it1)
    assert agree[well].mean() >= 0.97, agree[well].mean()
    assert dev[well].max() < 1e-4
