#!/usr/bin/env python
"""Dump K3 results (poses bits, iterations, status) for a fixed set of pool
pairs in several tiers -- compare two library builds bit for bit:
    RK_LIB=a.so python scripts/pose_dump.py out_a.npz; RK_LIB=b.so ... out_b.npz
    python scripts/pose_dump.py --compare out_a.npz out_b.npz"""
import os
import sys
from pathlib import Path

import numpy as np

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = {k: int((a[k] != b[k]).sum()) for k in a.files}
    print("mismatching entries:", bad)
    sys.exit(0 if not any(bad.values()) else 1)
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2112_02779_b200 as rk  # noqa: E402
from paper_2112_02779_b200 import pipeline, scenes  # noqa: E402
from paper_2112_02779_b200.range_image import normals_cross_batch  # noqa: E402

intr = scenes.ouster64()
pool = scenes.pair_pool_poses(300, seed=0)
src = pipeline.render_batch(intr, scenes.street_scene(), [b @ g for b, g in pool])
dst = pipeline.render_batch(intr, scenes.street_scene(), [b for b, _ in pool])
cfg = rk.RegistrationConfig()
surf = normals_cross_batch(intr, dst, strides=[s for s, _ in cfg.schedule])
out = {}
for tag, B, cl in (("x16", 4, None), ("x8", 12, None), ("x4", 30, None), ("x2", 100, None), ("wide", 200, None),
                   ("thr", 300, None), ("c1", 40, "0")):
    if cl is None:
        os.environ.pop("RK_ICP_CLUSTER", None)
    else:
        os.environ["RK_ICP_CLUSTER"] = cl
    idx = torch.arange(B, dtype=torch.int32, device="cuda")
    r = rk.register_batch(intr, src, dst, surf, idx, idx, config=cfg)
    out[f"{tag}_poses"] = r.poses.cpu().numpy().view(np.uint64)
    out[f"{tag}_iters"] = r.iterations.cpu().numpy()
    out[f"{tag}_status"] = r.status.cpu().numpy()
np.savez(sys.argv[1], **out)
print("saved", sys.argv[1])
