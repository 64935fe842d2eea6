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
(tests/test_gpu_bench_parity.py).

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
    print(f"{N_PAIRS} pairs in {time.time() - t0:.0f} s")
    out = {"pick": pick.astype(np.int64),
           "src_sha1": np.array([r["src_sha1"] for r in rows]),
           "dst_sha1": np.array([r["dst_sha1"] for r in rows]),
           "gt": np.stack([r["gt"] for r in rows])}
    for t in THREADS:
        out[f"t{t}/poses"] = np.stack([r[f"t{t}/poses"] for r in rows])
        out[f"t{t}/iters"] = np.array([r[f"t{t}/iters"] for r in rows], np.int32)
        out[f"t{t}/status"] = np.array([r[f"t{t}/status"] for r in rows], np.int32)
    out["t1/ncorr_flat"] = np.array([c for r in rows for c in r["ncorr"]], np.int64)
    out["t1/ncorr_len"] = np.array([len(r["ncorr"]) for r in rows], np.int64)
    out["numpy"] = np.array(np.__version__)
    np.savez_compressed(OUT / "c4_pool.npz", **out)
    p1 = out["t1/poses"]
    for t in THREADS[1:]:
        d = np.nanmax(np.abs(out[f"t{t}/poses"] - p1), axis=1)
        print(f"threads={t} vs 1: {(d > 1e-5).sum()} pairs > 1e-5, "
              f"{(out[f't{t}/iters'] != out['t1/iters']).sum()} iteration counts differ")
    print("wrote", OUT / "c4_pool.npz")


if __name__ == "__main__":
    main()
