import sys, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2112_02779_b200 as rk
from paper_2112_02779_b200 import pipeline, scenes
intr = scenes.ouster64()
pool = scenes.pair_pool_poses(2, seed=0)
src = pipeline.render_batch(intr, scenes.street_scene(), [b @ g for b, g in pool]).cpu().numpy()
dst = pipeline.render_batch(intr, scenes.street_scene(), [b for b, _ in pool]).cpu().numpy()
S, D = rk.RangeImage(src[0], intr), rk.RangeImage(dst[0], intr)
for _ in range(5): rk.register(S, D)
pr = cProfile.Profile(); pr.enable()
for _ in range(300): rk.register(S, D)
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(18)
