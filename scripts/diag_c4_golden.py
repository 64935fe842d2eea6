#!/usr/bin/env python
"""Per-pair view of the C4 reference goldens vs the GPU (MATH_NP / FAST):
the worst well-posed pairs with their iteration counts and per-iteration
correspondence counts.  python scripts/diag_c4_golden.py [np|fast]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2112_02779_b200 as rk  # noqa: E402
from paper_2112_02779_b200 import lidar_model as lm, pipeline, scenes  # noqa: E402

mode = {"np": lm.MATH_NP, "fast": lm.MATH_FAST, "cr": lm.MATH_CR}[sys.argv[1] if len(sys.argv) > 1 else "np"]
g = dict(np.load(ROOT / "tests" / "golden" / "c4_pool.npz"))
intr = scenes.ouster64()
pool = scenes.pair_pool_poses(2048, seed=0)
pick = g["pick"]
dst = pipeline.render_batch(intr, scenes.street_scene(), [pool[int(i)][0] for i in pick])
src = pipeline.render_batch(intr, scenes.street_scene(), [pool[int(i)][0] @ pool[int(i)][1] for i in pick])
with lm.math_mode(mode):
    res = rk.register_batch(intr, src, dst, with_stats=True)
P, it, stats = res.poses.cpu().numpy(), res.iterations.cpu().numpy(), res.stats.cpu().numpy()
ref, it1, gt = g["t1/poses"], g["t1/iters"], g["gt"]
well = np.linalg.norm(ref[:, 9:] - gt[:, 9:], axis=1) < 0.05
dev = np.abs(P - ref).max(axis=1)
off = np.concatenate([[0], np.cumsum(g["t1/ncorr_len"])])
order = np.argsort(-np.where(well, dev, -1))
for b in order[:5]:
    print(f"pair {b} (pool {pick[b]}): dev {dev[b]:.3g} iters gpu {it[b]} ref {it1[b]} "
          f"ref t8 dev {np.abs(g['t8/poses'][b] - ref[b]).max():.3g}")
    mine = stats[b, :it[b], :3]
    theirs = g["t1/ncorr_flat"][off[b]:off[b + 1]]
    print("  strides", mine[:, 0].astype(int).tolist())
    print("  gpu n  ", mine[:, 2].astype(int).tolist())
    print("  ref n  ", theirs.tolist())
