"""C4 goldens from the UNMODIFIED reference: 256 pairs of the benchmark's own
pool (``scenes.pair_pool_poses(2048, seed=0)``, the 256-pair parity subset
SURVEY §8(d) C4 asks for) rendered by ``synth.render_scene`` and registered by
``registration.register`` with the default config, at several shard counts:

* ``threads=1``  -- one shard, the schedule the oracle restates;
* ``threads=2, 4, 8`` -- the stride-1 level (n >= 40,000 points) split into
  that many float32 sgemm partials merged in float64
  (registration.py:252-260, 292-326); 8 = min(8, cores) is the reference's
  default on an 8+-core host (registration.py:361-366).

The reference's own disagreement between these runs (same inputs, same
numpy/OpenBLAS, only the float32 summation split differs) is the floor a
GPU kernel that also reorders float32 sums can be held to
(tests/test_gpu_bench_parity.py).  The shard count only splits the
stride-1 level, so a second floor covers every level: ``f64sum`` is the
reference with its float32 sgemm/sgemv normal-equation sums replaced by
float64 sums of the same float32 per-point terms (a monkeypatch of
_partial_normal_equations, used for this measurement only) -- how far the
reference's result depends on its own summation rounding, which at the
coarse levels is ~1e-5 relative (float32 over thousands of terms).

Images are not stored: the per-image SHA-1 of the reference's float32 bytes
is, and the GPU test re-renders them with ``rk_render`` and requires equal
hashes -- which is also the renderer's bit-exact parity check.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_c4.py
"""

from __future__ import annotations

import hashlib
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT.parent.parent))
sys.path.insert(0, str(OUT))

import numpy as np  # noqa: E402

import rangekit as rk  # noqa: E402  (the reference)
from rangekit.errors import DegenerateGeometry  # noqa: E402
from rangekit.range_image import compute_normal_map  # noqa: E402
from rangekit import registration  # noqa: E402
from rangekit.registration import RegistrationConfig, register  # noqa: E402
from rangekit.synth import render_scene  # noqa: E402

from make_golden import ref_intr, ref_pose, ref_scene  # noqa: E402
from paper_2112_02779_b200 import scenes  # noqa: E402  (input definitions only)

N_PAIRS = 256
THREADS = (1, 2, 4, 8)


def pick_pairs():
    """The C4 parity subset (test_gpu_bench_parity.py), first N_PAIRS."""
    return np.random.default_rng(2026).choice(2048, size=256, replace=False)[:N_PAIRS]


def sha(a: np.ndarray) -> str:
    return hashlib.sha1(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def _f64_sums(orig):
    """_partial_normal_equations with the SAME float32 per-point terms
    (J * w, r * w) summed in float64 instead of float32 sgemm/sgemv: the
    reference's formula without its own summation rounding."""
    def run(corr, pose, kernel_scale):
        out = orig(corr, pose, kernel_scale)
        n = out[0]
        if not n:
            return out
        moved = (corr.source @ pose.R.T + pose.t).astype(np.float32)
        nrm = np.asarray(corr.normal, dtype=np.float32)
        tgt = np.asarray(corr.target, dtype=np.float32)
        r = np.einsum("ij,ij->i", nrm, moved - tgt)
        J = np.empty((n, 6), np.float32)
        mx, my, mz = moved[:, 0], moved[:, 1], moved[:, 2]
        nx, ny, nz = nrm[:, 0], nrm[:, 1], nrm[:, 2]
        J[:, 0] = my * nz - mz * ny
        J[:, 1] = mz * nx - mx * nz
        J[:, 2] = mx * ny - my * nx
        J[:, 3:] = nrm
        w = registration.robust_weight32(r, np.float32(kernel_scale))
        Jw = (J * w[:, None]).astype(np.float64)
        H = Jw.T @ J.astype(np.float64)
        b = -((r * w).astype(np.float64) @ J.astype(np.float64))
        return n, H, b, out[3], out[4]
    return run


def one_pair_f64(n):
    """threads=1 with float64 normal-equation sums (see _f64_sums)."""
    intr = ref_intr(scenes.ouster64())
    scene = ref_scene(scenes.street_scene())
    i = int(pick_pairs()[n])
    base, g = scenes.pair_pool_poses(2048, seed=0)[i]
    dst = render_scene(scene, intr, ref_pose(base))
    src = render_scene(scene, intr, ref_pose(base @ g))
    orig = registration._partial_normal_equations
    registration._partial_normal_equations = _f64_sums(orig)
    try:
        res = register(src, dst, config=RegistrationConfig(threads=1), dst_normals=compute_normal_map(dst))
        return np.concatenate([res.pose.R.reshape(-1), res.pose.t]), res.iterations, 0 if res.converged else 1
    except DegenerateGeometry:
        return np.full(12, np.nan), -1, 2
    finally:
        registration._partial_normal_equations = orig


def one_pair(n):
    """Render and register pool pair ``pick_pairs()[n]`` with the reference
    (a worker process; the registrations run sequentially inside it)."""
    intr = ref_intr(scenes.ouster64())
    scene = ref_scene(scenes.street_scene())
    i = int(pick_pairs()[n])
    base, g = scenes.pair_pool_poses(2048, seed=0)[i]
    dst = render_scene(scene, intr, ref_pose(base))
    src = render_scene(scene, intr, ref_pose(base @ g))
    nrm = compute_normal_map(dst)
    row = dict(src_sha1=sha(src.data), dst_sha1=sha(dst.data), gt=g.as_row12())
    for t in THREADS:
        try:
            res = register(src, dst, config=RegistrationConfig(threads=t), dst_normals=nrm)
            row[f"t{t}/poses"] = np.concatenate([res.pose.R.reshape(-1), res.pose.t])
            row[f"t{t}/status"] = 0 if res.converged else 1
            row[f"t{t}/iters"] = res.iterations
            if t == 1:
                row["ncorr"] = [s.n_correspondences for s in res.stats]
        except DegenerateGeometry:
            row[f"t{t}/poses"] = np.full(12, np.nan)
            row[f"t{t}/status"] = 2
            row[f"t{t}/iters"] = -1
            if t == 1:
                row["ncorr"] = []
    return row


def main():
    from concurrent.futures import ProcessPoolExecutor
    pick = pick_pairs()
    t0 = time.time()
    with ProcessPoolExecutor(os.cpu_count() or 1) as ex:
        rows = list(ex.map(one_pair, range(N_PAIRS)))
        f64 = list(ex.map(one_pair_f64, range(N_PAIRS)))
    print(f"{N_PAIRS} pairs in {time.time() - t0:.0f} s")
    out = {"pick": pick.astype(np.int64),
           "src_sha1": np.array([r["src_sha1"] for r in rows]),
           "dst_sha1": np.array([r["dst_sha1"] for r in rows]),
           "gt": np.stack([r["gt"] for r in rows])}
    for t in THREADS:
        out[f"t{t}/poses"] = np.stack([r[f"t{t}/poses"] for r in rows])
        out[f"t{t}/iters"] = np.array([r[f"t{t}/iters"] for r in rows], np.int32)
        out[f"t{t}/status"] = np.array([r[f"t{t}/status"] for r in rows], np.int32)
    out["f64sum/poses"] = np.stack([r[0] for r in f64])
    out["f64sum/iters"] = np.array([r[1] for r in f64], np.int32)
    out["f64sum/status"] = np.array([r[2] for r in f64], np.int32)
    out["t1/ncorr_flat"] = np.array([c for r in rows for c in r["ncorr"]], np.int64)
    out["t1/ncorr_len"] = np.array([len(r["ncorr"]) for r in rows], np.int64)
    out["numpy"] = np.array(np.__version__)
    np.savez_compressed(OUT / "c4_pool.npz", **out)
    p1 = out["t1/poses"]
    well = np.linalg.norm(p1[:, 9:] - out["gt"][:, 9:], axis=1) < 0.05
    for t in [f"t{t}" for t in THREADS[1:]] + ["f64sum"]:
        d = np.nanmax(np.abs(out[f"{t}/poses"] - p1), axis=1)
        flip = (d > 1e-5) | (out[f"{t}/iters"] != out["t1/iters"])
        print(f"{t} vs threads=1: well-posed {int(flip[well].sum())}/{int(well.sum())} differ "
              f"(> 1e-5 or iterations), ill-posed {int(flip[~well].sum())}/{int((~well).sum())}")
    print("wrote", OUT / "c4_pool.npz")


if __name__ == "__main__":
    main()
