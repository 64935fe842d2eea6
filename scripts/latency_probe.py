#!/usr/bin/env python
"""register() latency from host arrays (the graph path) and the K3 kernel
alone for one pair, by cluster size (RK_ICP_CLUSTER) and math mode."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2112_02779_b200 as rk  # noqa: E402
from paper_2112_02779_b200 import lidar_model as lm, pipeline, scenes  # noqa: E402
from paper_2112_02779_b200.range_image import normals_cross_batch  # noqa: E402

intr = scenes.ouster64()
pool = scenes.pair_pool_poses(4, seed=0)
src = pipeline.render_batch(intr, scenes.street_scene(), [b @ g for b, g in pool])
dst = pipeline.render_batch(intr, scenes.street_scene(), [b for b, _ in pool])
sh, dh = src.cpu().numpy(), dst.cpu().numpy()
cfg = rk.RegistrationConfig()
surf = normals_cross_batch(intr, dst, strides=[s for s, _ in cfg.schedule])
for mode in ("np", "fast"):
    for cl in sys.argv[1:] or ["8", "16"]:
        os.environ["RK_ICP_CLUSTER"] = cl
        with lm.math_mode(lm.MATH_NP if mode == "np" else lm.MATH_FAST):
            rk.registration._pair_graphs.clear()
            idx = torch.zeros(1, dtype=torch.int32, device="cuda")
            for _ in range(3):
                r = rk.register_batch(intr, src, dst, surf, idx, idx, config=cfg)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                r = rk.register_batch(intr, src, dst, surf, idx, idx, config=cfg)
            e1.record()
            torch.cuda.synchronize()
            k_ms = e0.elapsed_time(e1) / 20
            for _ in range(3):
                rk.register(rk.RangeImage(sh[0], intr), rk.RangeImage(dh[0], intr))
            t = time.perf_counter()
            for k in range(30):
                res = rk.register(rk.RangeImage(sh[k % 4], intr), rk.RangeImage(dh[k % 4], intr))
            ms = (time.perf_counter() - t) / 30 * 1e3
            print(f"{mode} cluster {cl}: K3 {k_ms:.3f} ms, register() {ms:.3f} ms, "
                  f"pose0 {r.poses[0, 9].item():.9f} iters {r.iterations[0].item()}", flush=True)
