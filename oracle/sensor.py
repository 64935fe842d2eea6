"""Oracle: cylindrical sensor model (tables, projection, unprojection).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
``rangekit/lidar_model.py``; citations are to that file unless noted.
"""

from __future__ import annotations

import numpy as np

from .exactmath import asin_f32, atan2_f32

F32 = np.float32
TWO_PI = 2.0 * np.pi  # lidar_model.py:25

OK, OUT_OF_FOV, DEGENERATE = 0, 1, 2  # lidar_model.py:31-33


class Sensor:
    """Per-sensor tables exactly as the reference derives them.

    * inverse elevation LUT: K = factor*H uniform bins over the LUT span, each
      holding the nearest row (lowest row on ties)       -- lines 69-91
    * ray directions / receiver origins (float64, then float32 copies)
                                                          -- lines 138-179
    * field-of-view bounds widened by half a ray gap    -- lines 128-136
    """

    def __init__(self, width, height, receiver_radius, azimuth_lut, elevation_lut,
                 inv_factor=2):
        self.W = int(width)
        self.H = int(height)
        self.r0 = float(receiver_radius)
        self.az = np.asarray(azimuth_lut, dtype=np.float64).reshape(-1)
        self.el = np.asarray(elevation_lut, dtype=np.float64).reshape(-1)
        H, W = self.H, self.W

        lo_el, hi_el = float(self.el.min()), float(self.el.max())
        K = inv_factor * H
        centres = np.linspace(lo_el, hi_el, K)
        dist = np.abs(self.el[None, :] - centres[:, None])
        self.inv_rows = np.argmin(dist, axis=1).astype(np.int32)
        self.inv_lo, self.inv_hi = lo_el, hi_el

        # fov: one end is the smallest elevation; widen both ends by half the
        # spacing to the adjacent row
        if self.el[0] < self.el[-1]:
            gap_lo = abs(self.el[0] - self.el[1])
            gap_hi = abs(self.el[H - 1] - self.el[H - 2])
        else:
            gap_lo = abs(self.el[H - 1] - self.el[H - 2])
            gap_hi = abs(self.el[0] - self.el[1])
        self.fov = (float(self.el.min() - 0.5 * gap_lo), float(self.el.max() + 0.5 * gap_hi))

        col_angle = TWO_PI * np.arange(W) / W
        ray_theta = col_angle[None, :] + self.az[:, None]
        cphi = np.cos(self.el[:, None])
        self.dirs = np.empty((H, W, 3))
        self.dirs[..., 0] = np.cos(ray_theta) * cphi
        self.dirs[..., 1] = np.sin(ray_theta) * cphi
        self.dirs[..., 2] = np.sin(self.el)[:, None]
        self.origins = np.zeros((W, 3))
        self.origins[:, 0] = self.r0 * np.cos(col_angle)
        self.origins[:, 1] = self.r0 * np.sin(col_angle)
        self.dirs32 = self.dirs.astype(F32)
        self.origins32 = self.origins.astype(F32)
        self.az32 = self.az.astype(F32)
        self.el32 = self.el.astype(F32)

    @classmethod
    def from_intrinsics(cls, intr):
        """Build from any object with the LidarIntrinsics attribute names."""
        return cls(intr.width, intr.height, intr.receiver_radius, intr.azimuth_lut,
                   intr.elevation_lut, getattr(intr, "inv_factor", 2))

    # ------------------------------------------------------------ rows
    def row_lookup(self, phi):
        """Nearest-bin row (InverseElevationLut.lookup, lines 60-66).

        float32 phi keeps every step in float32 (numpy weak scalars)."""
        phi = np.asarray(phi)
        K = self.inv_rows.shape[0]
        scale = (K - 1) / (self.inv_hi - self.inv_lo)
        if phi.dtype == np.float32:
            pos = (phi - F32(self.inv_lo)) * F32(scale) + F32(0.5)
            pos = np.minimum(np.maximum(pos, F32(0)), F32(K - 1))
        else:
            pos = np.minimum(np.maximum((phi - self.inv_lo) * scale + 0.5, 0.0), K - 1.0)
        return self.inv_rows[pos.astype(np.int32)]

    def row_from_elevation(self, phi):
        """+-1 refinement, lowest row wins ties (lines 181-202)."""
        phi = np.asarray(phi)
        table = self.el32 if phi.dtype == np.float32 else self.el
        v0 = self.row_lookup(phi).astype(np.int32)
        cand = np.stack([np.maximum(v0 - 1, 0), v0, np.minimum(v0 + 1, self.H - 1)])
        err = np.abs(table[cand] - phi[None])
        # first index of the minimum error over (v-1, v, v+1)
        pick = np.argmin(err, axis=0)
        return np.take_along_axis(cand, pick[None], axis=0)[0].astype(np.int32)

    # ------------------------------------------------------------ projection
    def project_f32(self, points, math="numpy"):
        """Bulk float32 projection, ``project_many(single=True, refine=False)``
        (lines 262-344: 288-289 azimuth, 293-297 closed-form receiver, 311,
        315 elevation, 316 row, 319-321 column wrap, 338-344 status)."""
        p = np.asarray(points, dtype=F32)
        x, y, z = p[..., 0], p[..., 1], p[..., 2]
        W = self.W
        cols_per_rad = F32(W / TWO_PI)
        theta = atan2_f32(y, x, math)
        u_hat = np.where(theta < 0, theta + F32(TWO_PI), theta + F32(0.0)) * cols_per_rad
        r0 = F32(self.r0)
        if r0 > 0:
            rho2 = x * x + y * y
            degenerate = rho2 + z * z <= r0 * r0
            shrink = F32(1.0) - r0 / np.sqrt(np.maximum(rho2, F32(1e-30)))
            xc, yc = x * shrink, y * shrink
            r = np.sqrt(xc * xc + yc * yc + z * z)
        else:
            r = np.sqrt(x * x + y * y + z * z)
            degenerate = r <= 0
        q = np.clip(z / np.maximum(r, F32(1e-30)), F32(-1.0), F32(1.0))
        phi = asin_f32(q, math)
        v = self.row_from_elevation(phi)
        u = u_hat - cols_per_rad * self.az32[v]
        u = np.where(u < 0, u + F32(W), u)
        u = np.where(u >= W, u - F32(W), u)
        status = np.zeros(p.shape[:-1], dtype=np.int8)
        status[(phi < F32(self.fov[0])) | (phi > F32(self.fov[1]))] = OUT_OF_FOV
        status[degenerate] = DEGENERATE
        return u, v, r, status

    def project_f64(self, points, max_iters=3, tol=1e-4, refine=True):
        """Float64 iterative projection (lines 287-344, single=False path)."""
        p = np.asarray(points, dtype=np.float64)
        x, y, z = p[..., 0], p[..., 1], p[..., 2]
        W = self.W
        cpr = W / TWO_PI
        r0 = self.r0

        def wrap_angle(th):
            return (th + TWO_PI * (th < 0)) * cpr

        with np.errstate(invalid="ignore", divide="ignore"):
            u_hat = wrap_angle(np.arctan2(y, x))
            if r0 > 0.0:
                rho2 = x * x + y * y
                degenerate = rho2 + z * z <= r0 * r0
                xc, yc = x, y
                for _ in range(max_iters):
                    a = u_hat / cpr
                    xc = x - r0 * np.cos(a)
                    yc = y - r0 * np.sin(a)
                    u_new = wrap_angle(np.arctan2(yc, xc))
                    d = np.abs(u_new - u_hat)
                    d = np.minimum(d, W - d)
                    u_hat = u_new
                    live = d[~degenerate]
                    if live.size == 0 or live.max() < tol:
                        break
                r = np.sqrt(xc * xc + yc * yc + z * z)
            else:
                r = np.sqrt(x * x + y * y + z * z)
                degenerate = r <= 0.0
            phi = np.arcsin(np.clip(z / np.maximum(r, 1e-300), -1.0, 1.0))
            v = self.row_from_elevation(phi)
            u = u_hat - cpr * self.az[v]
            u = u + W * (u < 0)
            u = u - W * (u >= W)
            if r0 > 0.0 and refine:
                a = u / cpr
                xc = x - r0 * np.cos(a)
                yc = y - r0 * np.sin(a)
                r = np.sqrt(xc * xc + yc * yc + z * z)
                phi = np.arcsin(np.clip(z / np.maximum(r, 1e-300), -1.0, 1.0))
                v = self.row_from_elevation(phi)
                u = wrap_angle(np.arctan2(yc, xc)) - cpr * self.az[v]
                u = u + W * (u < 0)
                u = u - W * (u >= W)
        status = np.zeros(p.shape[:-1], dtype=np.int8)
        status[(phi < self.fov[0]) | (phi > self.fov[1])] = OUT_OF_FOV
        status[degenerate] = DEGENERATE
        return u, v.astype(np.int64), r, status

    # ------------------------------------------------------------ unprojection
    def unproject_image(self, rng):
        """p = r*dir + origin in float64 (range_image.py:129-133)."""
        r = np.asarray(rng, dtype=np.float32).astype(np.float64)
        return r[..., None] * self.dirs + self.origins[None, :, :]

    def unproject_pixels(self, v, u, r):
        """Flat-table gathers (range_image.py:160-167)."""
        flat = np.asarray(v) * self.W + np.asarray(u)
        r = np.asarray(r, dtype=np.float64)
        dirs = self.dirs.reshape(-1, 3)
        return r[:, None] * dirs[flat] + self.origins[np.asarray(u)]

    def unproject_many(self, u, v, r):
        """Analytic unprojection (lidar_model.py:236-250)."""
        u = np.asarray(u, dtype=np.float64)
        v = np.asarray(v, dtype=np.int64)
        r = np.asarray(r, dtype=np.float64)
        alpha = TWO_PI * u / self.W
        theta = alpha + self.az[v]
        phi = self.el[v]
        cphi = np.cos(phi)
        return np.stack([r * np.cos(theta) * cphi + self.r0 * np.cos(alpha),
                         r * np.sin(theta) * cphi + self.r0 * np.sin(alpha),
                         r * np.sin(phi) + np.zeros_like(u)], axis=-1)
