"""Oracle: projective point-to-plane ICP (association, normal equations, schedule).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
``rangekit/registration.py`` and the pose algebra of ``rangekit/se3.py``.
"""

from __future__ import annotations

import numpy as np

from .exactmath import rows_times_mat_t
from .image import points_at_stride
from .sensor import F32

EYE3 = np.eye(3)


# ---------------------------------------------------------------- SE(3) (se3.py)

def hat(w):
    return np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])


def so3_exp(omega):
    """Rodrigues (se3.py:22-31)."""
    omega = np.asarray(omega, dtype=float)
    th = np.linalg.norm(omega)
    if th < 1e-12:
        K = hat(omega)
        return EYE3 + K + 0.5 * (K @ K)
    K = hat(omega / th)
    return EYE3 + np.sin(th) * K + (1.0 - np.cos(th)) * (K @ K)


def se3_exp(xi):
    """Twist [omega, nu] -> (R, t) (se3.py:49-63)."""
    xi = np.asarray(xi, dtype=float).reshape(6)
    w, nu = xi[:3], xi[3:]
    R = so3_exp(w)
    th = np.linalg.norm(w)
    if th < 1e-12:
        V = EYE3 + 0.5 * hat(w)
    else:
        K = hat(w)
        V = EYE3 + (1.0 - np.cos(th)) / th ** 2 * K + (th - np.sin(th)) / th ** 3 * (K @ K)
    return R, V @ nu


def compose(a, b):
    """(Ra, ta) o (Rb, tb) (se3.py:65-67)."""
    return a[0] @ b[0], a[0] @ b[1] + a[1]


def orthonormality_defect(R):
    return float(np.linalg.norm(R.T @ R - EYE3))


def reorthonormalize(R):
    """Nearest rotation via SVD (se3.py:95-102)."""
    U, _, Vt = np.linalg.svd(R)
    Q = U @ Vt
    if np.linalg.det(Q) < 0:
        U[:, -1] = -U[:, -1]
        Q = U @ Vt
    return Q


# ---------------------------------------------------------------- association

def correspondences_f32(sensor, src_pts, dst_rng, dst_nrm, dst_valid, R, t, max_dist,
                        stride=1, math="numpy", fma="exact"):
    """Bulk float32 projective association (registration.py:117-187, single=True).

    Returns (sel, target f32 (M,3), normal f32 (M,3), moved32 (N,3)) where
    ``sel`` indexes the surviving source points (row order preserved).
    """
    src = np.asarray(src_pts, dtype=np.float64).reshape(-1, 3)
    W, H = sensor.W, sensor.H
    moved = rows_times_mat_t(src, R, t, mode=fma)
    m32 = moved.astype(F32)
    u, v, _, status = sensor.project_f32(m32, math=math)
    inv_s = F32(1.0 / stride)
    col = (u * inv_s + F32(0.5)).astype(np.int32) * stride
    col[col >= W] = 0
    row = (v.astype(F32) * inv_s + F32(0.5)).astype(np.int32) * stride
    ok = (status == 0) & (row >= 0) & (row < H)
    row = np.clip(row, 0, H - 1)
    flat = row * W + col
    rng = np.asarray(dst_rng, dtype=F32).reshape(-1)
    r_px = rng[flat]
    ok &= (r_px > 0) & np.asarray(dst_valid).reshape(-1)[flat]
    sel = np.flatnonzero(ok)
    fq, cq, rq = flat[sel], col[sel], r_px[sel]
    d32 = sensor.dirs32.reshape(-1, 3)
    o32 = sensor.origins32
    tgt = np.empty((sel.size, 3), dtype=F32)
    d2 = np.zeros(sel.size, dtype=F32)
    for c in range(3):
        tgt[:, c] = rq * d32[fq, c] + o32[cq, c]
        diff = m32[sel, c] - tgt[:, c]
        d2 = d2 + diff * diff
    keep = d2 <= F32(max_dist) * F32(max_dist)
    nrm = np.asarray(dst_nrm, dtype=F32).reshape(-1, 3)
    return sel[keep], tgt[keep], nrm[fq[keep]], m32


def correspondences_f64(sensor, src_pts, dst_rng, dst_nrm, dst_valid, R, t, max_dist,
                        stride=1, fma="exact"):
    """Float64 association (registration.py:117-187, single=False): iterative
    projection with refine, float64 targets.  Returns (sel, target, normal)."""
    src = np.asarray(src_pts, dtype=np.float64).reshape(-1, 3)
    W, H = sensor.W, sensor.H
    moved = rows_times_mat_t(src, R, t, mode=fma)
    u, v, _, status = sensor.project_f64(moved, refine=True)
    inv_s = 1.0 / stride
    col = (u * inv_s + 0.5).astype(np.int32) * stride
    col[col >= W] = 0
    row = (v.astype(np.float64) * inv_s + 0.5).astype(np.int32) * stride
    ok = (status == 0) & (row >= 0) & (row < H)
    row = np.clip(row, 0, H - 1)
    flat = row * np.int32(W) + col
    r_px = np.asarray(dst_rng, dtype=F32).reshape(-1)[flat]
    ok &= (r_px > 0) & np.asarray(dst_valid).reshape(-1)[flat]
    sel = np.flatnonzero(ok)
    fq, cq = flat[sel], col[sel]
    rq = r_px[sel].astype(np.float64)
    d64 = sensor.dirs.reshape(-1, 3)
    tgt = np.empty((sel.size, 3))
    d2 = np.zeros(sel.size)
    for c in range(3):
        tgt[:, c] = rq * d64[fq, c] + sensor.origins[cq, c]
        diff = moved[sel, c] - tgt[:, c]
        d2 = d2 + diff * diff
    keep = d2 <= max_dist * max_dist
    nrm = np.asarray(dst_nrm, dtype=F32).reshape(-1, 3)[fq[keep]].astype(np.float64)
    return sel[keep], tgt[keep], nrm


def normal_equations_f32(src_sel, tgt, nrm, R, t, kernel, fma="exact"):
    """Float32 shard contribution (registration.py:329-358).

    Returns (n, H f64 6x6, b f64 6, cost, sumsq).  H and b are formed in
    float32 with the same BLAS calls as the reference (sgemm / sgemv), so on
    the reference host they match bit for bit; the CUDA reduction agrees to
    float32 reassociation error.
    """
    n = src_sel.shape[0]
    if n == 0:
        return 0, np.zeros((6, 6)), np.zeros(6), 0.0, 0.0
    m = rows_times_mat_t(src_sel, R, t, mode=fma).astype(F32)
    q = tgt.astype(F32)
    nv = nrm.astype(F32)
    r = np.einsum("ij,ij->i", nv, m - q)
    J = np.empty((n, 6), dtype=F32)
    J[:, 0] = m[:, 1] * nv[:, 2] - m[:, 2] * nv[:, 1]
    J[:, 1] = m[:, 2] * nv[:, 0] - m[:, 0] * nv[:, 2]
    J[:, 2] = m[:, 0] * nv[:, 1] - m[:, 1] * nv[:, 0]
    J[:, 3:] = nv
    k32 = F32(kernel)
    w = F32(1.0) / np.sqrt(F32(1.0) + (r / k32) ** 2)
    Jw = J * w[:, None]
    Hm = (Jw.T @ J).astype(np.float64)
    b = (-(r * w) @ J).astype(np.float64)
    cost = float(kernel ** 2 * np.sum(F32(1.0) / w - F32(1.0), dtype=np.float64))
    sumsq = float(r @ r)
    return n, Hm, b, cost, sumsq


# ---------------------------------------------------------------- schedule

DEFAULT_SCHEDULE = ((4, 20), (2, 20), (1, 10))


class DegenerateGeometryError(Exception):
    pass


def _shard_bounds(n, shards):
    """registration.py:292-296: one shard below 40,000 points or 1 thread."""
    if shards <= 1 or n < 40_000:
        return [(0, n)]
    edges = np.linspace(0, n, shards + 1).astype(int)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]


def _normal_equations_sharded(sensor, src, dst_rng, dst_nrm, dst_valid, R, t, gate, stride, kern,
                              shards, pool, math, fma):
    """_accumulate_normal_equations (registration.py:299-326): per-shard
    association + float32 partial systems (on the thread pool), merged in
    shard order in float64."""
    def run(ab):
        a, b = ab
        sel, tgt, nrm, _ = correspondences_f32(sensor, src[a:b], dst_rng, dst_nrm, dst_valid,
                                               R, t, gate, stride, math=math, fma=fma)
        return normal_equations_f32(src[a:b][sel], tgt, nrm, R, t, kern, fma=fma)
    parts = list(pool.map(run, shards)) if pool is not None and len(shards) > 1 else [run(s) for s in shards]
    n = sum(p[0] for p in parts)
    Hm, b, cost, sumsq = np.zeros((6, 6)), np.zeros(6), 0.0, 0.0
    for ni, Hi, bi, ci, si in parts:
        if ni:
            Hm += Hi
            b += bi
            cost += ci
            sumsq += si
    return n, Hm, b, cost, sumsq


def register(sensor, src_rng, dst_rng, dst_nrm, dst_valid, R0=None, t0=None, *,
             kernel_scale=0.5, max_dist=0.5, schedule=DEFAULT_SCHEDULE, rot_eps=1e-4,
             trans_eps=1e-4, clip_min=0.0, clip_max=np.inf, min_corr=6,
             scale_with_stride=True, math="numpy", fma="exact", threads=1):
    """Coarse-to-fine ICP (registration.py:237-289).  threads > 1 shards the
    levels of >= 40,000 points over a thread pool exactly as the reference
    does (its RANGEKIT_THREADS / RegistrationConfig.threads); threads=1 is
    the single-shard schedule the goldens were made with.

    Returns dict(R, t, converged, stats=[(stride, it, n, cost, rmse)], degenerate).
    """
    from concurrent.futures import ThreadPoolExecutor
    R = EYE3.copy() if R0 is None else np.asarray(R0, dtype=float).copy()
    t = np.zeros(3) if t0 is None else np.asarray(t0, dtype=float).copy()
    stats = []
    pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None
    try:
        return _register_levels(sensor, src_rng, dst_rng, dst_nrm, dst_valid, R, t, stats, pool, threads,
                                kernel_scale, max_dist, schedule, rot_eps, trans_eps, clip_min, clip_max,
                                min_corr, scale_with_stride, math, fma)
    finally:
        if pool is not None:
            pool.shutdown(wait=False)


def _register_levels(sensor, src_rng, dst_rng, dst_nrm, dst_valid, R, t, stats, pool, threads,
                     kernel_scale, max_dist, schedule, rot_eps, trans_eps, clip_min, clip_max,
                     min_corr, scale_with_stride, math, fma):
    for stride, iters in schedule:
        level = float(stride) if scale_with_stride else 1.0
        gate = max_dist * level
        kern = kernel_scale * level
        src = points_at_stride(sensor, src_rng, stride, clip_min, clip_max)
        shards = _shard_bounds(src.shape[0], threads if pool else 1)
        for it in range(iters):
            n, Hm, b, cost, sumsq = _normal_equations_sharded(sensor, src, dst_rng, dst_nrm, dst_valid,
                                                              R, t, gate, stride, kern, shards, pool,
                                                              math, fma)
            if n < min_corr:
                return dict(R=R, t=t, converged=False, stats=stats, degenerate=False)
            if np.linalg.cond(Hm) > 1e12:
                return dict(R=R, t=t, converged=False, stats=stats, degenerate=True)
            xi = np.linalg.solve(Hm, b)
            R, t = compose(se3_exp(xi), (R, t))
            if orthonormality_defect(R) > 1e-12:
                R = reorthonormalize(R)
            stats.append((stride, it, n, cost, float(np.sqrt(sumsq / n))))
            if np.linalg.norm(xi[:3]) < rot_eps and np.linalg.norm(xi[3:]) < trans_eps:
                break
    return dict(R=R, t=t, converged=True, stats=stats, degenerate=False)


def centroid_translation(src_pts, dst_pts):
    """initial_translation_by_centroids (registration.py:96-102)."""
    return np.asarray(dst_pts, float).mean(axis=0) - np.asarray(src_pts, float).mean(axis=0)
