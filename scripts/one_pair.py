#!/usr/bin/env python
"""One register_batch launch of one pair (the latency mode), repeated: a
small target for ncu captures of K3's cluster kernel."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2112_02779_b200 as rk  # noqa: E402
from paper_2112_02779_b200 import pipeline, scenes  # noqa: E402
from paper_2112_02779_b200.range_image import normals_cross_batch  # noqa: E402

intr = scenes.ouster64()
pool = scenes.pair_pool_poses(1, seed=0)
src = pipeline.render_batch(intr, scenes.street_scene(), [b @ g for b, g in pool])
dst = pipeline.render_batch(intr, scenes.street_scene(), [b for b, _ in pool])
cfg = rk.RegistrationConfig()
surf = normals_cross_batch(intr, dst, strides=[s for s, _ in cfg.schedule])
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    rk.register_batch(intr, src, dst, surf, config=cfg)
torch.cuda.synchronize()
