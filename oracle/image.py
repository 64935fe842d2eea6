"""Oracle: range-image operations (point clouds, pyramid views, cross and PCA
normals, cloud -> image z-buffer).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
``rangekit/range_image.py``; citations are to that file.
"""

from __future__ import annotations

import numpy as np

from .sensor import OK, OUT_OF_FOV, DEGENERATE, F32


def valid_clip_mask(rng, clip_min=0.0, clip_max=np.inf):
    """r > 0 and clip_min <= r <= clip_max, compared in float32 (lines 140, 152)."""
    r = np.asarray(rng, dtype=F32)
    return (r > 0) & (r >= F32(clip_min)) & (r <= F32(clip_max))


def to_point_cloud(sensor, rng, clip_min=0.0, clip_max=np.inf):
    """Valid, clipped pixels in row-major order, unprojected in float64 (136-143)."""
    r = np.asarray(rng, dtype=F32)
    v, u = np.nonzero(valid_clip_mask(r, clip_min, clip_max))
    rr = r[v, u].astype(np.float64)
    return rr[:, None] * sensor.dirs[v, u] + sensor.origins[u]


def stride_indices(rng, stride, clip_min=0.0, clip_max=np.inf):
    """Row-major (v, u) base pixels of the stride-s view that survive the mask
    (StridedView 69-116 + points_at_stride 146-157)."""
    r = np.asarray(rng, dtype=F32)
    view = r[::stride, ::stride]
    vi, ui = np.nonzero(valid_clip_mask(view, clip_min, clip_max))
    return vi * stride, ui * stride


def points_at_stride(sensor, rng, stride, clip_min=0.0, clip_max=np.inf):
    r = np.asarray(rng, dtype=F32)
    v, u = stride_indices(r, stride, clip_min, clip_max)
    return sensor.unproject_pixels(v, u, r[v, u].astype(np.float64))


def normals_cross(sensor, rng):
    """Cross-product normals (221-240) in the op order SURVEY Appendix A1 pins.

    Returns (vectors float32 (H,W,3), valid bool (H,W)).
    """
    r = np.asarray(rng, dtype=F32)
    P = sensor.unproject_image(r)
    ok0 = r > 0
    right = np.roll(P, -1, axis=1)
    right_ok = np.roll(ok0, -1, axis=1)
    down = np.zeros_like(P)
    down[:-1] = P[1:]
    down_ok = np.zeros_like(ok0)
    down_ok[:-1] = ok0[1:]
    a = right - P
    b = down - P
    c = np.empty_like(P)
    c[..., 0] = a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1]
    c[..., 1] = a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2]
    c[..., 2] = a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]
    nn = np.sqrt((c[..., 0] * c[..., 0] + c[..., 1] * c[..., 1]) + c[..., 2] * c[..., 2])
    valid = ok0 & right_ok & down_ok & (nn > 1e-12)
    with np.errstate(invalid="ignore", divide="ignore"):
        n = c / nn[..., None]
    facing = (n[..., 0] * P[..., 0] + n[..., 1] * P[..., 1]) + n[..., 2] * P[..., 2]
    n = np.where((facing > 0)[..., None], -n, n)
    n[~valid] = 0.0
    return n.astype(F32), valid


def from_point_cloud(sensor, points, max_iters=3, tol=1e-4):
    """z-buffer projection of a cloud into a fresh image (170-194).

    Returns (image float32 (H,W), dict(kept, collisions, out_of_fov, degenerate)).
    """
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    H, W = sensor.H, sensor.W
    buf = np.full(H * W, np.inf)
    stats = dict(kept=0, collisions=0, out_of_fov=0, degenerate=0)
    if pts.shape[0]:
        u, v, r, st = sensor.project_f64(pts, max_iters=max_iters, tol=tol)
        good = st == OK
        stats["out_of_fov"] = int(np.count_nonzero(st == OUT_OF_FOV))
        stats["degenerate"] = int(np.count_nonzero(st == DEGENERATE))
        col = np.mod(np.floor(u[good] + 0.5).astype(np.int64), W)
        flat = v[good] * W + col
        np.minimum.at(buf, flat, r[good])
        n_in = int(np.count_nonzero(good))
        n_pix = int(np.unique(flat).shape[0]) if n_in else 0
        stats["kept"] = n_pix
        stats["collisions"] = n_in - n_pix
    buf[~np.isfinite(buf)] = 0.0
    return buf.reshape(H, W).astype(F32), stats


def normals_pca(sensor, rng, radius=2, disc_abs=0.3, disc_rel=0.05):
    """Windowed-PCA normals (243-283): float64 window sums in the (dv, du)
    order, covariance, numpy eigh's smallest eigenvector, sensor-facing.

    Returns (vectors float32 (H,W,3), valid bool (H,W)).
    """
    r32 = np.asarray(rng, dtype=F32)
    P = sensor.unproject_image(r32)
    valid = r32 > 0
    r = r32.astype(np.float64)
    H, W = r.shape
    count = np.zeros((H, W))
    s1 = np.zeros((H, W, 3))
    s2 = np.zeros((H, W, 3, 3))
    thresh = disc_abs + disc_rel * r
    for dv in range(-radius, radius + 1):
        for du in range(-radius, radius + 1):
            q = np.roll(P, -du, axis=1)
            qv = np.roll(valid, -du, axis=1)
            qr = np.roll(r, -du, axis=1)
            if dv:
                q2 = np.zeros_like(q)
                qv2 = np.zeros_like(qv)
                qr2 = np.zeros_like(qr)
                if dv > 0:
                    q2[:-dv], qv2[:-dv], qr2[:-dv] = q[dv:], qv[dv:], qr[dv:]
                else:
                    q2[-dv:], qv2[-dv:], qr2[-dv:] = q[:dv], qv[:dv], qr[:dv]
                q, qv, qr = q2, qv2, qr2
            w = (valid & qv & (np.abs(qr - r) <= thresh)).astype(np.float64)
            count += w
            s1 += w[..., None] * q
            s2 += w[..., None, None] * (q[..., :, None] * q[..., None, :])
    ok = valid & (count >= 3)
    n = np.zeros((H, W, 3))
    if np.any(ok):
        c = count[ok][:, None]
        mean = s1[ok] / c
        cov = s2[ok] / c[..., None] - mean[:, :, None] * mean[:, None, :]
        n[ok] = np.linalg.eigh(cov)[1][:, :, 0]
    flip = np.sum(n * P, axis=-1) > 0
    n[flip] = -n[flip]
    n[~ok] = 0.0
    return n.astype(F32), ok
