"""Probe: register consecutive C5 extended-street frames in chunks (timing,
iteration counts, statuses) -- used to bisect a pathological pair.
    python scripts/odometry_probe.py F lo hi [chunk]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2112_02779_b200 as rk  # noqa: E402
from paper_2112_02779_b200 import pipeline, scenes  # noqa: E402
from paper_2112_02779_b200.range_image import normals_cross_batch  # noqa: E402

intr = scenes.os128()
F, lo0, hi0 = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
chunk = int(sys.argv[4]) if len(sys.argv) > 4 else 100
traj = scenes.street_trajectory(F, seed=0, step_m=0.5, jitter=float(__import__('os').environ.get('JITTER', '0.0002')))
frames = pipeline.render_batch(intr, scenes.extended_street_scene(0.5 * F + 30.0), traj)
cfg = rk.RegistrationConfig()
surf = normals_cross_batch(intr, frames, strides=[s for s, _ in cfg.schedule])
torch.cuda.synchronize()
for lo in range(lo0, hi0, chunk):
    hi = min(lo + chunk, hi0, F - 1)
    ps = torch.arange(lo + 1, hi + 1, dtype=torch.int32, device='cuda')
    res = rk.register_batch(intr, frames, frames, surf, ps, ps - 1, config=cfg)
    t = time.perf_counter()
    torch.cuda.synchronize()
    it = res.iterations.cpu().numpy()
    st = res.status.cpu().numpy()
    print(lo, hi, round(time.perf_counter() - t, 3), 's iters max', it.max(), 'status',
          np.bincount(st, minlength=4), flush=True)
