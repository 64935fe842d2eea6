"""Seeded float32 inputs for the numpy-exact transcendental parity test
(shared by make_golden_svml.py and tests/test_gpu_numpy_exact.py)."""

import numpy as np

N_ATAN2 = 4_000_000
N_ASIN = 4_000_000


def atan2_inputs(n=N_ATAN2):
    """(y, x): LiDAR-like coordinates over four decades, plus axes, zeros and
    signed zeros (SVML's scalar path)."""
    g = np.random.default_rng(20261019)
    scale = g.choice(np.array([1e-3, 0.1, 1.0, 30.0, 300.0]), size=(2, n))
    y = (g.normal(size=n) * scale[0]).astype(np.float32)
    x = (g.normal(size=n) * scale[1]).astype(np.float32)
    k = n // 100
    y[:k] = 0.0
    x[k:2 * k] = 0.0
    y[2 * k:3 * k] = -0.0
    x[3 * k:3 * k + k // 2] = -0.0
    y[4 * k:5 * k] = x[4 * k:5 * k]             # |y| == |x| (the k1 boundary)
    y[5 * k:6 * k] = -x[5 * k:6 * k]
    return y, x


def asin_inputs(n=N_ASIN):
    """z / r over [-1, 1]: uniform, the LiDAR band |q| < 0.5, near +-1 and
    the 0.5 branch boundary."""
    g = np.random.default_rng(20261020)
    q = np.concatenate([g.uniform(-1.0, 1.0, n // 2), g.uniform(-0.45, 0.45, n // 4),
                        g.uniform(0.999, 1.0, n // 8) * g.choice([-1.0, 1.0], n // 8),
                        g.uniform(0.4999, 0.5001, n - n // 2 - n // 4 - n // 8)])
    q = q.astype(np.float32)
    q[:8] = np.array([0.0, -0.0, 1.0, -1.0, 0.5, -0.5, 1e-30, -1e-38], np.float32)
    return q
