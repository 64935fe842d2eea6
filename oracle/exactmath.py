"""Exact float64 FMA and correctly-rounded float32 transcendentals (oracle helpers).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference computes every ``(n,3) @ (3,3)`` transform with OpenBLAS dgemm
(registration.py:146, sdf_volume.py:159-160, se3.py:79).  On the survey host
that kernel evaluates ``fma(p2, M2j, fma(p1, M1j, p0 * M0j))`` (SURVEY
Appendix A2).  numpy has no fused multiply-add ufunc, so ``fma`` below emulates
it exactly: Dekker's exact product, Knuth's TwoSum, and the
round-to-odd construction of Boldo & Melquiond ("Emulation of FMA and correctly
rounded sums: proved algorithms using rounding to odd", IEEE TC 2008,
Algorithm 5.4), which is correctly rounded in binary64 barring over/underflow.
"""

from __future__ import annotations

import numpy as np

_SPLITTER = 134217729.0  # 2**27 + 1 (Veltkamp split for binary64)


def _two_sum(a, b):
    s = a + b
    bv = s - a
    av = s - bv
    return s, (a - av) + (b - bv)


def _split(a):
    c = _SPLITTER * a
    hi = c - (c - a)
    return hi, a - hi


def _two_prod(a, b):
    p = a * b
    ah, al = _split(a)
    bh, bl = _split(b)
    err = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    return p, err


def _round_to_odd_sum(a, b):
    """RO(a + b): the odd neighbour of RN(a+b) whenever the sum is inexact."""
    s, e = _two_sum(a, b)
    bits = s.view(np.int64)
    inexact = (e != 0.0) & ((bits & 1) == 0)
    toward = np.where(e > 0.0, np.inf, -np.inf)
    return np.where(inexact, np.nextafter(s, toward), s)


def fma(a, b, c):
    """Correctly rounded a*b + c, elementwise, float64."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    a, b, c = np.broadcast_arrays(a, b, c)
    with np.errstate(over="ignore", invalid="ignore"):
        uh, ul = _two_prod(a, b)
        th, tl = _two_sum(c, uh)
        v = _round_to_odd_sum(tl, ul)
        out = th + v
    # exact zero products / non-finite inputs: fall back to the plain expression
    plain = a * b + c
    bad = ~np.isfinite(out) | ~np.isfinite(uh)
    return np.where(bad, plain, out)


def rows_times_mat_t(points, M, t=None, mode="exact"):
    """``points @ M.T (+ t)`` with the pinned OpenBLAS op order.

    out_j = fma(p2, M[j,2], fma(p1, M[j,1], p0 * M[j,0])) (+ t_j, separate add).
    ``mode="blas"`` uses numpy's matmul (the reference's literal call).
    """
    points = np.asarray(points, dtype=np.float64)
    M = np.asarray(M, dtype=np.float64).reshape(3, 3)
    if mode == "blas":
        out = points @ M.T
        return out if t is None else out + np.asarray(t, dtype=np.float64)
    p0, p1, p2 = points[..., 0], points[..., 1], points[..., 2]
    # a single row goes through dgemv, whose kernel starts from the middle
    # term: fma(p2, M2j, fma(p0, M0j, p1*M1j)) (measured on the survey host)
    single = points.ndim == 1 or points.shape[0] == 1
    cols = []
    for j in range(3):
        if single:
            acc = p1 * M[j, 1]
            acc = fma(p0, M[j, 0], acc)
        else:
            acc = p0 * M[j, 0]
            acc = fma(p1, M[j, 1], acc)
        acc = fma(p2, M[j, 2], acc)
        if t is not None:
            acc = acc + float(t[j])
        cols.append(acc)
    return np.stack(cols, axis=-1)


_svml_lib = None


def _svml():
    """oracle/svml_emu.c (numpy's SVML float32 arctan2 / arcsin restated in C),
    compiled on first use into oracle/_build/ with the host's gcc."""
    global _svml_lib
    if _svml_lib is None:
        import ctypes
        import subprocess
        from pathlib import Path
        here = Path(__file__).resolve().parent
        src = here / "svml_emu.c"
        so = here / "_build" / "libsvml_emu.so"
        if not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
            so.parent.mkdir(exist_ok=True)
            subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", str(src), "-o",
                            str(so), "-lm"], check=True)
        lib = ctypes.CDLL(str(so))
        lib.svml_atan2f_n.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_long]
        lib.svml_asinf_n.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_long]
        tab = np.fromfile(here.parent / "paper_2112_02779_b200" / "data" / "vrsqrt14.u16", dtype="<u2")
        _svml_lib = (lib, np.ascontiguousarray(tab))
    return _svml_lib


def svml_atan2(y, x):
    """numpy's AVX-512 float32 arctan2, host-independent (svml_emu.c)."""
    lib, _ = _svml()
    y, x = np.broadcast_arrays(np.asarray(y, dtype=np.float32), np.asarray(x, dtype=np.float32))
    y, x = np.ascontiguousarray(y), np.ascontiguousarray(x)
    out = np.empty(y.shape, np.float32)
    lib.svml_atan2f_n(y.ctypes.data, x.ctypes.data, out.ctypes.data, y.size)
    return out


def svml_asin(q):
    """numpy's AVX-512 float32 arcsin, host-independent (svml_emu.c)."""
    lib, tab = _svml()
    q = np.ascontiguousarray(np.asarray(q, dtype=np.float32))
    out = np.empty(q.shape, np.float32)
    lib.svml_asinf_n(q.ctypes.data, tab.ctypes.data, out.ctypes.data, q.size)
    return out


def atan2_f32(y, x, math="numpy"):
    """math: "numpy" (the host's own np.arctan2, what the reference runs),
    "svml" (numpy's AVX-512 result on any host), "cr" (correctly rounded)."""
    y = np.asarray(y, dtype=np.float32)
    x = np.asarray(x, dtype=np.float32)
    if math == "numpy":
        return np.arctan2(y, x)
    if math == "svml":
        return svml_atan2(y, x)
    return np.arctan2(y.astype(np.float64), x.astype(np.float64)).astype(np.float32)


def asin_f32(q, math="numpy"):
    q = np.asarray(q, dtype=np.float32)
    if math == "numpy":
        return np.arcsin(q)
    if math == "svml":
        return svml_asin(q)
    return np.arcsin(q.astype(np.float64)).astype(np.float32)
