#!/usr/bin/env python
"""K3 time per register_batch call for mid-size batches under the launcher's
choice, the throughput kernel (RK_ICP_WIDE=0) and forced x2 / x4 clusters."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2112_02779_b200 as rk  # noqa: E402
from paper_2112_02779_b200 import pipeline, scenes  # noqa: E402
from paper_2112_02779_b200.range_image import normals_cross_batch  # noqa: E402

intr = scenes.ouster64()
pool = scenes.pair_pool_poses(256, seed=0)
src = pipeline.render_batch(intr, scenes.street_scene(), [b @ g for b, g in pool])
dst = pipeline.render_batch(intr, scenes.street_scene(), [b for b, _ in pool])
cfg = rk.RegistrationConfig()
if len(sys.argv) > 1 and sys.argv[1] == "fast":  # the FAST kernels' crossovers
    from paper_2112_02779_b200 import lidar_model as lm
    lm.set_default_math(lm.MATH_FAST)
surf = normals_cross_batch(intr, dst, strides=[s for s, _ in cfg.schedule])


def run(B, env, reps=5):
    for k in ("RK_ICP_WIDE", "RK_ICP_CLUSTER"):
        os.environ.pop(k, None)
    os.environ.update(env)
    idx = (torch.arange(B, dtype=torch.int32, device="cuda") % 256).to(torch.int32)
    for _ in range(2):
        rk.register_batch(intr, src, dst, surf, idx, idx, config=cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        rk.register_batch(intr, src, dst, surf, idx, idx, config=cfg)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


for B in (100, 149, 200, 296, 297, 400, 444):
    r = {"auto": run(B, {}), "thr": run(B, {"RK_ICP_WIDE": "0"}), "x2": run(B, {"RK_ICP_CLUSTER": "2"}),
         "x4": run(B, {"RK_ICP_CLUSTER": "4"})}
    print(f"B={B}: " + ", ".join(f"{k} {v:.2f} ms" for k, v in r.items()), flush=True)
