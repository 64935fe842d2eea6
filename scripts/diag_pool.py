import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2112_02779_b200 as rk
from paper_2112_02779_b200 import lidar_model as lm, pipeline, scenes
from oracle import icp as oicp, image as oimg, sensor as osens
intr = scenes.ouster64(); S = osens.Sensor.from_intrinsics(intr)
street = scenes.street_scene(); pool = scenes.pair_pool_poses(2048, seed=0)
pick = np.random.default_rng(2026).choice(len(pool), size=48, replace=False)
src = pipeline.render_batch(intr, street, [pool[i][0] @ pool[i][1] for i in pick])
dst = pipeline.render_batch(intr, street, [pool[i][0] for i in pick])
out = {}
for mode in ("fast", "cr"):
    lm.set_default_math(lm.MATH_CR if mode == "cr" else lm.MATH_FAST)
    r = rk.register_batch(intr, src, dst, with_stats=True)
    out[mode] = (r.poses.cpu().numpy(), r.iterations.cpu().numpy(), r.status.cpu().numpy())
lm.set_default_math(lm.MATH_FAST)
sh, dh = src.cpu().numpy(), dst.cpu().numpy()
gt = np.stack([pool[i][1].as_row12() for i in pick])
for b in range(48):
    vec, valid = oimg.normals_cross(S, dh[b])
    ref = oicp.register(S, sh[b], dh[b], vec, valid, math="cr", fma="exact")
    line = []
    for mode in ("fast", "cr"):
        P, it, st = out[mode]
        dR = np.abs(P[b, :9].reshape(3, 3) - ref["R"]).max(); dt = np.abs(P[b, 9:] - ref["t"]).max()
        line.append(f"{mode}: dR {dR:.1e} dt {dt:.1e} it {it[b]}/{len(ref['stats'])} st {st[b]}")
    gterr = np.linalg.norm(out['fast'][0][b, 9:] - gt[b, 9:])
    bad = any(float(x.split('dR ')[1].split()[0]) > 1e-5 for x in line)
    if bad or b < 3:
        print(b, f"gt_err {gterr:.3f} conv {ref['converged']}", " | ".join(line))
