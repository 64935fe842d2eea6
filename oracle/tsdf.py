"""Oracle: sparse 16^3-block TSDF (activation, integration, trilinear query).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
``rangekit/sdf_volume.py``; citations are to that file.

The grid is a plain ``dict[(i,j,k)] -> (tsdf f32 (16,16,16), weight f32 (16,16,16))``.
"""

from __future__ import annotations

import numpy as np

from .exactmath import rows_times_mat_t
from .sensor import F32

EDGE = 16  # line 22
VOXELS = EDGE ** 3
# C-order local voxel indices, z fastest (line 26)
LOCAL = np.stack(np.meshgrid(np.arange(EDGE), np.arange(EDGE), np.arange(EDGE),
                             indexing="ij"), axis=-1).reshape(-1, 3).astype(np.int64)
CHUNK_BLOCKS = max(1, 600_000 // VOXELS)  # line 142: 146 blocks per task


def block_keys_for_points(points, radius, extent):
    """All block keys whose cube meets [p - radius, p + radius] (lines 82-106)."""
    p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    if p.shape[0] == 0:
        return set()
    lo = np.floor((p - radius) / extent).astype(np.int64)
    hi = np.floor((p + radius) / extent).astype(np.int64)
    span = hi - lo
    smax = span.max(axis=0)
    found = []
    for a in range(int(smax[0]) + 1):
        for b in range(int(smax[1]) + 1):
            for c in range(int(smax[2]) + 1):
                off = np.array([a, b, c])
                rows = np.all(span >= off, axis=1)
                found.append(lo[rows] + off)
    uniq = np.unique(np.concatenate(found), axis=0)
    return set(map(tuple, uniq.tolist()))


def activate(grid, points, radius, extent):
    """Insert zeroed blocks for every touched key; return the touched set."""
    touched = block_keys_for_points(points, radius, extent)
    for k in touched:
        if k not in grid:
            grid[k] = (np.zeros((EDGE,) * 3, F32), np.zeros((EDGE,) * 3, F32))
    return touched


def _chunk_centres(keys, R_inv, t_inv, voxel, fma="exact", lone=None):
    """Sensor-frame voxel centres of a chunk of blocks (lines 157-161).

    base (float64, one row per block) and the rotated local lattice are rounded
    to float32 separately and summed in float32.  A chunk
    of ONE block goes through dgemv, whose FMA order differs (exactmath);
    ``lone`` overrides whether this chunk is such a lone block (None: decided
    by the chunk's own length).
    """
    kb = np.asarray(keys, dtype=np.float64).reshape(-1, 3) * (EDGE * voxel)
    if lone is False and kb.shape[0] == 1:
        base = rows_times_mat_t(np.repeat(kb, 2, axis=0), R_inv, t_inv, mode=fma)[:1]
    else:
        base = rows_times_mat_t(kb, R_inv, t_inv, mode=fma)
    off = rows_times_mat_t((LOCAL + 0.5) * voxel, R_inv, None, mode=fma).astype(F32)
    return (base.astype(F32)[:, None, :] + off[None, :, :]).reshape(-1, 3)


def integrate(grid, sensor, rng, R, t, keys, voxel, trunc, max_weight=100.0,
              free_space=True, clip_min=0.0, clip_max=np.inf, math="numpy", fma="exact",
              touched=None, threads=1):
    """Projective running-average update of the given blocks (lines 116-186).

    (R, t) maps the frame into the world; its inverse is formed with numpy as
    the reference does (se3.py:72-74).  Returns the number of updated voxels.

    ``touched``: integrate only ``keys`` but with the arithmetic each block
    gets inside this larger touched set (the reference chunks the sorted set
    in 146-block tasks; only a lone last block is computed differently), so a
    sample of blocks can be checked without integrating the whole frame.
    ``threads`` > 1 runs the chunks on a thread pool as the reference does
    (sdf_volume.py:144-151); the result does not depend on it.
    """
    R = np.asarray(R, dtype=float)
    t = np.asarray(t, dtype=float)
    R_inv = R.T
    t_inv = -R_inv @ t
    order = sorted(keys)
    img = np.asarray(rng, dtype=F32)
    W = sensor.W
    tau = F32(trunc)
    lone_key = None
    if touched is None:
        chunks = [order[i0:i0 + CHUNK_BLOCKS] for i0 in range(0, len(order), CHUNK_BLOCKS)]
    else:
        full = sorted(touched)
        lone_key = full[-1] if len(full) % CHUNK_BLOCKS == 1 else None
        # every block but the lone one in multi-row chunks
        rest = [k for k in order if k != lone_key]
        chunks = [rest[i0:i0 + CHUNK_BLOCKS] for i0 in range(0, len(rest), CHUNK_BLOCKS)]
        if lone_key is not None and lone_key in set(order):
            chunks.append([lone_key])

    def one(part):
        lone = None if touched is None else (part == [lone_key])
        x = _chunk_centres(part, R_inv, t_inv, voxel, fma=fma, lone=lone)
        u, v, r, status = sensor.project_f32(x, math=math)
        col = (u + F32(0.5)).astype(np.int32)
        col[col == W] = 0
        px = img.reshape(-1)[v * np.int32(W) + col]
        ok = (status == 0) & (px > 0) & (px >= F32(clip_min)) & (px <= F32(clip_max))
        ok &= r <= F32(clip_max)
        d = px - r
        ok &= d >= -tau
        if not free_space:
            ok &= d <= tau
        d = np.minimum(d, tau)
        ts = np.stack([grid[k][0].reshape(-1) for k in part]).reshape(-1)
        ws = np.stack([grid[k][1].reshape(-1) for k in part]).reshape(-1)
        with np.errstate(invalid="ignore"):
            ts_new = np.where(ok, (ws * ts + d) / (ws + F32(1.0)), ts)
        ws_new = np.where(ok, np.minimum(ws + F32(1.0), F32(max_weight)), ws)
        for j, k in enumerate(part):
            grid[k] = (ts_new[j * VOXELS:(j + 1) * VOXELS].reshape((EDGE,) * 3),
                       ws_new[j * VOXELS:(j + 1) * VOXELS].reshape((EDGE,) * 3))
        return int(np.count_nonzero(ok))

    if threads > 1 and len(chunks) > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=threads) as ex:
            updated = sum(ex.map(one, chunks))
    else:
        updated = sum(one(part) for part in chunks)
    return updated


def integrate_cloud_frame(grid, sensor, rng, R, t, voxel, trunc, max_weight=100.0,
                          free_space=True, radius=None, clip_min=0.0, clip_max=np.inf,
                          math="numpy", fma="exact", threads=1):
    """activate + integrate for one posed frame (lines 198-210)."""
    from .image import to_point_cloud

    radius = trunc if radius is None else radius
    pts = to_point_cloud(sensor, rng, clip_min, clip_max)
    world = rows_times_mat_t(pts, R, t, mode=fma)
    keys = activate(grid, world, radius, EDGE * voxel)
    n = integrate(grid, sensor, rng, R, t, keys, voxel, trunc, max_weight, free_space,
                  clip_min, clip_max, math=math, fma=fma, threads=threads)
    return keys, n


def query_many(grid, pts, voxel):
    """Trilinear (sdf, weight, observed) over the 8 enclosing centres (lines 221-265)."""
    pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    g = pts / voxel - 0.5
    base = np.floor(g).astype(np.int64)
    frac = g - base
    n = pts.shape[0]
    sdf = np.zeros(n)
    wt = np.zeros(n)
    ok = np.ones(n, dtype=bool)
    for cx in (0, 1):
        for cy in (0, 1):
            for cz in (0, 1):
                off = np.array([cx, cy, cz])
                idx = base + off
                cw = np.prod(np.where(off == 1, frac, 1.0 - frac), axis=1)
                d = np.zeros(n, dtype=F32)
                w = np.zeros(n, dtype=F32)
                found = np.zeros(n, dtype=bool)
                bk = np.floor_divide(idx, EDGE)
                loc = idx - bk * EDGE
                for i in range(n):
                    blk = grid.get(tuple(int(q) for q in bk[i]))
                    if blk is not None:
                        d[i] = blk[0][tuple(loc[i])]
                        w[i] = blk[1][tuple(loc[i])]
                        found[i] = True
                ok &= found & (w > 0)
                sdf += cw * d
                wt += cw * w
    return sdf, wt, ok
