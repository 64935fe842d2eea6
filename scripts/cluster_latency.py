"""K3 latency mode: one pair per CTA vs one pair per cluster of 2/4/8 CTAs
(RK_ICP_CLUSTER), time per register_batch call and the pose difference
against the single-CTA result, by batch size.  Diagnostic."""
import os, sys, time
import torch
sys.path.insert(0, '.')
import paper_2112_02779_b200 as rk
from paper_2112_02779_b200 import pipeline, scenes
from paper_2112_02779_b200.range_image import normals_cross_batch
intr = scenes.ouster64(); street = scenes.street_scene()
pool = scenes.pair_pool_poses(160, seed=0)
src = pipeline.render_batch(intr, street, [b @ g for b, g in pool]); dst = pipeline.render_batch(intr, street, [b for b, _ in pool])
cfg = rk.RegistrationConfig()
surf = normals_cross_batch(intr, dst, strides=[s for s, _ in cfg.schedule])


def run(B, cl, reps=10):
    if cl is None:
        os.environ.pop("RK_ICP_CLUSTER", None)  # the launcher's own choice
    else:
        os.environ["RK_ICP_CLUSTER"] = str(cl)
    idx = torch.arange(B, dtype=torch.int32, device='cuda')
    for _ in range(2): res = rk.register_batch(intr, src, dst, surf, idx, idx, config=cfg)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): res = rk.register_batch(intr, src, dst, surf, idx, idx, config=cfg)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3, res


for B in (1, 4, 8, 9, 18, 33, 37, 50, 66, 67, 74, 99, 148):
    base_ms, base = run(B, 0)
    line = [f"B={B}: 1 CTA {base_ms:.3f} ms"]
    for cl in (2, 4, 8, 16, None):
        ms, r = run(B, cl)
        dp = (r.poses - base.poses).abs().max().item()
        same = bool((r.status == base.status).all().item())
        dit = (r.iterations - base.iterations).abs().max().item() if hasattr(r, "iterations") else -1
        line.append(f"cl{cl or 'auto'} {ms:.3f} ms (|dpose| {dp:.1e}, status {'=' if same else '!='}, |dit| {dit})")
    print("; ".join(line), flush=True)
