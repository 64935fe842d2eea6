import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2112_02779_b200 as rk
from paper_2112_02779_b200 import pipeline, scenes, registration as reg
intr = scenes.ouster64()
pool = scenes.pair_pool_poses(2, seed=0)
src = pipeline.render_batch(intr, scenes.street_scene(), [b @ g for b, g in pool]).cpu().numpy()
dst = pipeline.render_batch(intr, scenes.street_scene(), [b for b, _ in pool]).cpu().numpy()
S, D = rk.RangeImage(src[0], intr), rk.RangeImage(dst[0], intr)
for _ in range(5): rk.register(S, D)
plan = next(iter(reg._pair_graphs.values()))
N = 50
t0 = time.perf_counter()
for _ in range(N): rk.register(S, D)
t_all = (time.perf_counter() - t0) / N
t0 = time.perf_counter()
for _ in range(N):
    plan.h_src.numpy()[...] = src[0]; plan.h_dst.numpy()[...] = dst[0]
t_copy = (time.perf_counter() - t0) / N
t0 = time.perf_counter()
for _ in range(N):
    plan.graph.replay(); torch.cuda.current_stream().synchronize()
t_replay = (time.perf_counter() - t0) / N
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N): plan.graph.replay()
e1.record(); torch.cuda.synchronize()
print(f"register() {t_all*1e3:.3f} ms; staging copies {t_copy*1e3:.3f} ms; replay+sync {t_replay*1e3:.3f} ms; graph device time {e0.elapsed_time(e1)/N:.3f} ms")
