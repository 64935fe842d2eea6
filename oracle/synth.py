"""Oracle: analytic ray caster used to make parity-test inputs.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
``rangekit/synth.py``.  Primitives are plain tuples so the package's scene
definitions (``paper_2112_02779_b200.scenes``) can be passed straight in:

* ("plane", normal(3), offset)
* ("sphere", centre(3), radius)
* ("box", centre(3), size(3), rotation 3x3 or None)
"""

from __future__ import annotations

import numpy as np

MIN_HIT = 1e-9  # synth.py:19


def _plane(o, d, normal, offset):
    n = np.asarray(normal, float)
    den = d @ n
    with np.errstate(divide="ignore", invalid="ignore"):
        t = (offset - o @ n) / den
    t[(np.abs(den) < 1e-15) | (t <= MIN_HIT)] = np.inf
    return t


def _sphere(o, d, centre, radius):
    oc = o - np.asarray(centre, float)
    b = np.sum(oc * d, axis=-1)
    q = np.sum(oc * oc, axis=-1) - radius ** 2
    disc = b * b - q
    hit = disc >= 0
    s = np.sqrt(np.where(hit, disc, 0.0))
    near, far = -b - s, -b + s
    t = np.where(near > MIN_HIT, near, far)
    return np.where(hit & (t > MIN_HIT), t, np.inf)


def _box(o, d, centre, size, rot):
    R = np.eye(3) if rot is None else np.asarray(rot, float)
    half = 0.5 * np.asarray(size, float)
    lo_ = (o - np.asarray(centre, float)) @ R
    dl = d @ R
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / dl
        ta = (-half - lo_) * inv
        tb = (half - lo_) * inv
    par = np.abs(dl) < 1e-15
    enter = np.where(par, -np.inf, np.minimum(ta, tb))
    leave = np.where(par, np.inf, np.maximum(ta, tb))
    enter = np.where(par & ~(np.abs(lo_) <= half), np.inf, enter)
    t_in = enter.max(axis=-1)
    t_out = leave.min(axis=-1)
    t = np.where(t_in > MIN_HIT, t_in, t_out)
    return np.where((t_in > t_out) | (t <= MIN_HIT), np.inf, t)


def render(sensor, scene, R=None, t=None, noise_std=0.0, seed=None):
    """Nearest positive hit along every exact sensor ray (synth.py:108-134)."""
    H, W = sensor.H, sensor.W
    R = np.eye(3) if R is None else np.asarray(R, float)
    t = np.zeros(3) if t is None else np.asarray(t, float)
    d = sensor.dirs.reshape(-1, 3) @ R.T
    o = np.broadcast_to(sensor.origins[None], (H, W, 3)).reshape(-1, 3) @ R.T + t
    best = np.full(H * W, np.inf)
    for prim in scene:
        kind = prim[0]
        if kind == "plane":
            hit = _plane(o, d, prim[1], prim[2])
        elif kind == "sphere":
            hit = _sphere(o, d, prim[1], prim[2])
        elif kind == "box":
            hit = _box(o, d, prim[1], prim[2], prim[3] if len(prim) > 3 else None)
        else:
            raise ValueError(kind)
        np.minimum(best, hit, out=best)
    if noise_std > 0.0:
        g = np.random.default_rng(seed)
        m = np.isfinite(best)
        best[m] = np.maximum(best[m] + g.normal(0.0, noise_std, int(m.sum())), 0.0)
    best[~np.isfinite(best)] = 0.0
    return best.reshape(H, W).astype(np.float32)
