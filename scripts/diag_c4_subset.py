"""Per-pair diagnostic of the C4 256-pair parity subset: GPU (FAST, or CR=1)
vs the oracle; prints the well-posed pairs outside 1e-5 / equal iterations."""
import sys, os
sys.path.insert(0, '.')
sys.argv = ['x']
import numpy as np
sys.path.insert(0, "tests"); import test_gpu_bench_parity as T
import torch
import paper_2112_02779_b200 as rk
from paper_2112_02779_b200 import pipeline, scenes
intr = scenes.ouster64(); street = scenes.street_scene()
pool = scenes.pair_pool_poses(2048, seed=0)
pick = np.random.default_rng(2026).choice(len(pool), size=256, replace=False)
src = pipeline.render_batch(intr, street, [pool[i][0] @ pool[i][1] for i in pick])
dst = pipeline.render_batch(intr, street, [pool[i][0] for i in pick])
from paper_2112_02779_b200 import lidar_model as lm
MATH = lm.MATH_CR if os.environ.get('CR') else None
res = rk.register_batch(intr, src, dst, with_stats=True, math=MATH)
poses = res.poses.cpu().numpy(); iters = res.iterations.cpu().numpy()
src_h, dst_h = src.cpu().numpy(), dst.cpu().numpy()
gt = np.stack([pool[i][1].as_row12() for i in pick])
import multiprocessing as mp
from concurrent.futures import ProcessPoolExecutor
with ProcessPoolExecutor(16, mp_context=mp.get_context("fork")) as ex:
    refs = list(ex.map(T._oracle_pair, [(src_h[b], dst_h[b]) for b in range(256)]))
for b in range(256):
    R, t = poses[b, :9].reshape(3, 3), poses[b, 9:]
    rR, rt, rn = refs[b]
    ok = np.linalg.norm(rt - gt[b, 9:]) < 0.05
    dR, dt = np.abs(R - rR).max(), np.abs(t - rt).max()
    if ok and not (dR < 1e-5 and dt < 1e-5 and iters[b] == rn):
        st = res.stats[b, :iters[b]].cpu().numpy()
        print(b, pick[b], 'dR %.2e dt %.2e iters gpu %d ref %d' % (dR, dt, iters[b], rn), 'levels', [int(x) for x in st[:, 0]][-12:])
