"""register_batch time and throughput vs batch size (latency mode for
batches <= 2 pairs per SM; RK_ICP_WIDE=0 disables it).  Diagnostic."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2112_02779_b200 as rk
from paper_2112_02779_b200 import pipeline, scenes
intr = scenes.ouster64(); street = scenes.street_scene()
pool = scenes.pair_pool_poses(512, seed=0)
src = pipeline.render_batch(intr, street, [b @ g for b, g in pool]); dst = pipeline.render_batch(intr, street, [b for b, _ in pool])
from paper_2112_02779_b200.range_image import normals_cross_batch
cfg = rk.RegistrationConfig()
surf = normals_cross_batch(intr, dst, strides=[s for s, _ in cfg.schedule])
for B in (1, 64, 148, 200, 296, 400, 512):
    idx = torch.arange(B, dtype=torch.int32, device='cuda')
    for _ in range(2): rk.register_batch(intr, src, dst, surf, idx, idx, config=cfg)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): rk.register_batch(intr, src, dst, surf, idx, idx, config=cfg)
    torch.cuda.synchronize(); ms = (time.perf_counter() - t) / 5 * 1e3
    print(B, round(ms, 3), 'ms', round(B / ms * 1e3), 'reg/s')
