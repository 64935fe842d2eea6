"""Batched device pipelines behind the drop-in API: the callers the reference's
CLI runs in Python loops (cli.py:248-328 odometry / eval-reg pair sweeps,
cli.py:267-283 integrate) expressed as a few launches over device buffers.

* ``render_batch``   -- synthetic inputs on the device (synth.py:108-134, N4)
* ``odometry``       -- cli.py:248-263 frame-to-frame registration of a whole
  sequence as ONE register_batch launch + the host pose prefix product
* ``odometry_integrate`` -- C2 end to end: odometry, then the sequence
  integrated at the estimated poses
* ``eval_registration`` -- cli.py:294-328 ``cmd_eval_reg``: every sampled
  (i, i+d) pair of a sequence registered in ONE batched launch, scored
  against the ground-truth relative poses (the registration CSV rows)
* ``integrate_sequence`` -- activate + integrate F posed frames into one grid
  with no host synchronisation between frames
* ``shard`` / ``gather_poses`` -- one-process-per-GPU partitioning of
  independent pairs: contiguous slices, no data-path collective
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .trace import nvtx
from . import lidar_model as lm
from .distributed import all_gather_varsize, shard  # noqa: F401  (re-exported)
from .sdf_volume import VoxelBlockGrid
from .range_image import RangeImage, normals_cross_batch, to_point_cloud
from .registration import RegistrationConfig, initial_translation_by_centroids, register_batch
from .se3 import RigidTransform

_KIND = {"plane": 0, "sphere": 1, "box": 2}


def encode_scene(prims) -> np.ndarray:
    """Scene tuples (see scenes.py) -> (n, 16) float64 rows for rk_render."""
    rows = np.zeros((len(prims), 16))
    for i, p in enumerate(prims):
        rows[i, 0] = _KIND[p[0]]
        if p[0] == "plane":
            rows[i, 1:4] = p[1]
            rows[i, 4] = p[2]
        elif p[0] == "sphere":
            rows[i, 1:4] = p[1]
            rows[i, 4] = p[2]
        else:
            rows[i, 1:4] = p[1]
            rows[i, 4:7] = p[2]
            R = np.eye(3) if len(p) < 4 or p[3] is None else np.asarray(p[3], float)
            rows[i, 7:16] = R.reshape(-1)
    return rows


def poses_to_rows(poses) -> np.ndarray:
    return np.stack([p.as_row12() for p in poses]) if poses else np.zeros((0, 12))


def render_batch(intr: lm.LidarIntrinsics, scene, poses):
    """(B, H, W) float32 device range images of ``scene`` seen from each
    world-from-sensor pose."""
    prims = nat.to_dev(encode_scene(scene), np.float64)
    P = nat.to_dev(poses_to_rows(poses), np.float64)
    B = len(poses)
    out = nat.empty((B, intr.height, intr.width), np.float32)
    if B:
        nat.call("rk_render", lm.device_sensor(intr), nat.ptr(prims), prims.shape[0], nat.ptr(P), B,
                 nat.ptr(out), nat.stream_ptr())
    return out


def _check_frames(intr, frames):
    t = nat.torch()
    if not (nat.is_tensor(frames) and frames.is_cuda and frames.dtype == t.float32 and frames.ndim == 3
            and tuple(frames.shape[1:]) == (intr.height, intr.width)):
        raise ValueError(f"frames must be an (F, {intr.height}, {intr.width}) float32 CUDA tensor")


@nvtx("integrate_sequence")
def integrate_sequence(grid: VoxelBlockGrid, intr: lm.LidarIntrinsics, frames, poses_w,
                       inv_w=None, clip_min: float = 0.0, clip_max: float = np.inf,
                       radius: float | None = None, updated=None, graph: bool = False):
    """integrate_cloud_frame over F device frames, fully asynchronous.

    frames: (F, H, W) float32 device tensor; poses_w: (F, 12) float64 device
    world-from-frame rows; inv_w: (F, 12) their inverses formed on the host
    with numpy (as the reference's integrate() does) -- computed if None.
    Returns the device int64 counter of updated voxels.  The caller must size
    the grid (``grid.reserve``) and may check ``grid.info()`` for overflow.

    The activation of frame f+1 (side stream) overlaps the integration of
    frame f.  graph=True records the 4*F launches once as a CUDA graph (keyed
    by the buffers) and replays it on later calls with the same buffers: the
    frame stamps live on the device, so a replay is an exact re-run.
    """
    _check_frames(intr, frames)
    if tuple(poses_w.shape) != (frames.shape[0], 12) or poses_w.dtype != nat.torch().float64:
        raise ValueError("poses_w must be an (F, 12) float64 tensor")
    h = grid._prepare()
    sensor = lm.device_sensor(intr)
    radius = grid.truncation if radius is None else radius
    own_inv, own_upd = inv_w is None, updated is None
    if own_inv:
        host = nat.to_host(poses_w)
        inv_w = nat.to_dev(np.stack([RigidTransform(r[:9].reshape(3, 3), r[9:]).inverse().as_row12()
                                     for r in host]), np.float64)
    if own_upd:
        updated = nat.zeros((1,), np.int64)
    cmin, cmax = float(np.float32(clip_min)), float(np.float32(clip_max))
    math = lm.default_math()

    frames = frames.contiguous()
    poses_w = poses_w.contiguous()
    inv_w = inv_w.contiguous()

    def issue(inv, upd):
        # activation of frame f+1 overlaps the integration of frame f
        nat.call("rk_grid_integrate_frames", h, sensor, nat.ptr(frames), int(frames.shape[0]),
                 nat.ptr(poses_w), nat.ptr(inv), float(radius), cmin, cmax, math,
                 nat.ptr(upd), nat.stream_ptr())

    if not graph:
        issue(inv_w, updated)
    else:
        # graphs live on the grid (dropped when its tables are reallocated).
        # Buffers this function allocates itself (inverse poses, counter) are
        # owned by the cache entry and refilled per call, so they do not key
        # the cache: repeated calls replay one graph instead of recording a
        # new one per call.
        key = (sensor, frames.data_ptr(), tuple(frames.shape), poses_w.data_ptr(),
               None if own_inv else inv_w.data_ptr(), None if own_upd else updated.data_ptr(),
               float(radius), cmin, cmax, math)
        ent = grid._graphs.get(key)
        if ent is None:
            torch = nat.torch()
            ent = dict(inv=inv_w, upd=updated, g=torch.cuda.CUDAGraph())
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(ent["g"], stream=side, capture_error_mode="thread_local"):
                issue(ent["inv"], ent["upd"])
            torch.cuda.current_stream().wait_stream(side)
            grid.cache_graph(key, ent)
        else:
            if own_inv:
                ent["inv"].copy_(inv_w)
            if own_upd:
                ent["upd"].zero_()
        ent["g"].replay()
        updated = ent["upd"].clone() if own_upd else updated
    grid.blocks._bump()
    return updated


@nvtx("odometry")
def odometry(intr: lm.LidarIntrinsics, frames, config: RegistrationConfig = RegistrationConfig(),
             init: str = "identity", with_stats: bool = False):
    """Frame-to-frame odometry over a (F, H, W) float32 device sequence
    (cli.py:248-263 ``cmd_odometry``): frame k is registered to frame k-1
    from the identity (or, init="centroid", the centroid translation of the
    two clouds, cli.py:257-258) and world_k = world_{k-1} @ pose_k, world_0 =
    identity.  The F-1 pairs are independent, so they run as
    ONE register_batch launch over a surfel pyramid of the sequence; only the
    prefix product runs on the host, with the reference's own numpy
    composition (se3.py:69-71), so the chain rounds exactly as cmd_odometry's.

    Returns (world poses: list of F RigidTransform, BatchResult of the F-1
    relative registrations, or None when F < 2).
    """
    t = nat.torch()
    _check_frames(intr, frames)
    F = int(frames.shape[0])
    if init not in ("identity", "centroid"):
        raise ValueError("init must be 'identity' or 'centroid'")
    world = [RigidTransform.identity()]
    if F < 2:
        return world, None
    frames = frames.contiguous()
    dev = nat.device()
    pair_src = t.arange(1, F, dtype=t.int32, device=dev)
    pair_dst = t.arange(0, F - 1, dtype=t.int32, device=dev)
    inits = None
    if init == "centroid":
        clouds = [to_point_cloud(RangeImage(frames[k], intr)) for k in range(F)]
        inits = nat.to_dev(np.stack([initial_translation_by_centroids(clouds[k], clouds[k - 1]).as_row12()
                                     for k in range(1, F)]), np.float64)
    surf = normals_cross_batch(intr, frames, strides=[s for s, _ in config.schedule])
    res = register_batch(intr, frames, frames, surf, pair_src, pair_dst, inits, config,
                         with_stats=with_stats)
    rel = nat.to_host(res.poses)
    for k in range(F - 1):
        world.append(world[-1] @ RigidTransform(rel[k, :9].reshape(3, 3), rel[k, 9:]))
    return world, res


@nvtx("odometry_integrate")
def odometry_integrate(grid: VoxelBlockGrid, intr: lm.LidarIntrinsics, frames,
                       config: RegistrationConfig = RegistrationConfig(), init: str = "identity",
                       clip_min: float = 0.0, clip_max: float = np.inf, graph: bool = False):
    """C2 end to end (cli.py:248-283 odometry then integrate): estimate the
    sequence's trajectory and integrate every frame at its estimated pose.
    Returns (world poses, BatchResult, device int64 updated-voxel counter)."""
    world, res = odometry(intr, frames, config, init)
    poses_w = nat.to_dev(poses_to_rows(world), np.float64)
    inv_w = nat.to_dev(np.stack([p.inverse().as_row12() for p in world]), np.float64)
    updated = integrate_sequence(grid, intr, frames, poses_w, inv_w, clip_min=clip_min,
                                 clip_max=clip_max, graph=graph)
    return world, res, updated


REGISTRATION_CSV_HEADER = ("frame_distance,pair_index,rot_err_rad,trans_err_m,"
                           "converged,iters,runtime_ms")   # io_formats.py:368-369


def rotation_error(R, R_gt) -> float:
    """Geodesic angle arccos((trace(R R_gt^T) - 1) / 2) (eval_metrics.py:16-21)."""
    c = (np.trace(np.asarray(R, float) @ np.asarray(R_gt, float).T) - 1.0) / 2.0
    return float(np.arccos(np.clip(c, -1.0, 1.0)))


def translation_error(t, t_gt) -> float:
    """||t - t_gt|| in metres (eval_metrics.py:24-26)."""
    return float(np.linalg.norm(np.asarray(t, float) - np.asarray(t_gt, float)))


def sample_pairs(n_frames: int, frame_distance: int, count: int, seed=None):
    """count seeded (i, i + d) pairs without replacement when possible
    (eval_metrics.py:57-70, same generator calls, so the same pairs)."""
    from .errors import EmptyInput
    if frame_distance < 1:
        raise ValueError("frame distance must be >= 1")
    n_valid = n_frames - frame_distance
    if n_valid < 1:
        raise EmptyInput(f"no frame pairs at distance {frame_distance} in {n_frames} frames")
    if count >= n_valid:
        starts = np.arange(n_valid)
    else:
        starts = np.sort(np.random.default_rng(seed).choice(n_valid, size=count, replace=False))
    return [(int(i), int(i + frame_distance)) for i in starts]


@nvtx("eval_registration")
def eval_registration(intr: lm.LidarIntrinsics, frames, gt_poses, distances, pairs: int,
                      seed: int = 0, config: RegistrationConfig = RegistrationConfig(),
                      init: str = "identity"):
    """``cmd_eval_reg`` (cli.py:294-328) over a (F, H, W) device sequence:
    for each frame distance d, ``sample_pairs(F, d, pairs, seed + d)``; pair
    (i, j) registers frame j to frame i (init identity or centroid) and is
    scored against gt[i]^-1 @ gt[j].  All pairs of all distances run as ONE
    register_batch launch over one surfel pyramid of the sequence (the
    reference runs them on a thread pool, one register() each).

    Returns the CSV rows (d, pair_index, rot_err_rad, trans_err_m, converged,
    iters, runtime_ms); runtime_ms is the batch's wall time divided by the
    number of pairs (the amortised per-pair cost of the batched launch)."""
    import time
    t = nat.torch()
    _check_frames(intr, frames)
    F = int(frames.shape[0])
    if len(gt_poses) != F:
        raise ValueError("gt_poses must hold one pose per frame")
    jobs = []
    for d in distances:
        for k, (i, j) in enumerate(sample_pairs(F, int(d), pairs, seed=seed + int(d))):
            jobs.append((int(d), k, i, j))
    if not jobs:
        return []
    frames = frames.contiguous()
    dev = nat.device()
    t.cuda.synchronize()
    t0 = time.perf_counter()
    pair_dst = t.tensor([i for _, _, i, _ in jobs], dtype=t.int32, device=dev)
    pair_src = t.tensor([j for _, _, _, j in jobs], dtype=t.int32, device=dev)
    inits = None
    if init == "centroid":
        clouds = {}
        for f in {x for _, _, i, j in jobs for x in (i, j)}:
            clouds[f] = to_point_cloud(RangeImage(frames[f], intr))
        inits = nat.to_dev(np.stack([initial_translation_by_centroids(clouds[j], clouds[i]).as_row12()
                                     for _, _, i, j in jobs]), np.float64)
    elif init != "identity":
        raise ValueError("init must be 'identity' or 'centroid'")
    surf = normals_cross_batch(intr, frames, strides=[s for s, _ in config.schedule])
    res = register_batch(intr, frames, frames, surf, pair_src, pair_dst, inits, config)
    poses = nat.to_host(res.poses)
    status = nat.to_host(res.status)
    iters = nat.to_host(res.iterations)
    ms = 1e3 * (time.perf_counter() - t0) / len(jobs)
    rows = []
    for b, (d, k, i, j) in enumerate(jobs):
        rel_gt = gt_poses[i].inverse() @ gt_poses[j]
        R, tt = poses[b, :9].reshape(3, 3), poses[b, 9:]
        rows.append((d, k, rotation_error(R, rel_gt.R), translation_error(tt, rel_gt.t),
                     int(status[b] == 0), int(iters[b]), round(ms, 3)))
    return rows


def write_registration_csv(path, rows) -> None:
    """io_formats.py:373-378."""
    with open(path, "w", encoding="utf-8") as f:
        f.write(REGISTRATION_CSV_HEADER + "\n")
        for r in rows:
            f.write(",".join(str(x) for x in r) + "\n")


# launches issued per call (the bench's gpu_launches accounting)
LAUNCHES_PER_FRAME = 4     # begin (reset + count), activate, assign, integrate
LAUNCHES_CLEAR = 2         # k_clear_blocks, k_clear_counters (+2 memsets)


def clear_grid(grid: VoxelBlockGrid):
    nat.call("rk_grid_clear", grid._prepare(), nat.stream_ptr())
    grid.blocks._bump()


def gather_poses(local_poses, world: int):
    """All-gather per-rank (n_i, 12) pose slices (rank order) -- the only
    cross-rank traffic of a sharded ICP batch."""
    return local_poses if world == 1 else all_gather_varsize(local_poses)
