"""End-to-end use of the drop-in API on one B200: a synthetic 64x1024 street
sequence -> frame-to-frame ICP odometry -> TSDF integration at the estimated
poses -> marching cubes -> PLY, i.e. the reference CLI's
``odometry`` + ``integrate`` + ``mesh`` commands (cli.py:248-291) as three
batched calls.

    python examples/odometry_reconstruct.py [--frames 100] [--out street.ply]
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2112_02779_b200 as rk  # noqa: E402  (drop-in for `import rangekit as rk`)
from paper_2112_02779_b200 import io_formats, pipeline, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=100)
    ap.add_argument("--voxel", type=float, default=0.05)
    ap.add_argument("--out", default="street.ply")
    args = ap.parse_args()

    import torch
    intr = scenes.ouster64()
    truth = scenes.street_trajectory(args.frames, seed=0)
    frames = pipeline.render_batch(intr, scenes.street_scene(), truth)   # (F, 64, 1024) on the GPU
    torch.cuda.synchronize()

    grid = rk.VoxelBlockGrid(voxel_size=args.voxel, capacity=65536)
    t0 = time.perf_counter()
    world, rel, updated = pipeline.odometry_integrate(grid, intr, frames, clip_max=30.0)
    n_upd = int(updated.item())
    t1 = time.perf_counter()
    mesh = rk.extract_mesh(grid)
    t2 = time.perf_counter()
    io_formats.write_ply(args.out, mesh)

    drift = max(np.linalg.norm(w.t - (truth[0].inverse() @ p).t) for w, p in zip(world, truth))
    print(f"{args.frames} frames: odometry + TSDF {1e3 * (t1 - t0):.1f} ms "
          f"({args.frames / (t1 - t0):.0f} frames/s), {n_upd} voxel updates, "
          f"max drift {drift:.3f} m")
    print(f"marching cubes {1e3 * (t2 - t1):.1f} ms: {mesh.n_vertices} vertices, "
          f"{mesh.n_triangles} triangles -> {args.out}")


if __name__ == "__main__":
    main()
