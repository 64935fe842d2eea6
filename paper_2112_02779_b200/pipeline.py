"""Batched device pipelines behind the drop-in API: the callers the reference's
CLI runs in Python loops (cli.py:248-328 odometry / eval-reg pair sweeps,
cli.py:267-283 integrate) expressed as a few launches over device buffers.

* ``render_batch``   -- synthetic inputs on the device (synth.py:108-134, N4)
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
    h = grid._prepare()
    sensor = lm.device_sensor(intr)
    radius = grid.truncation if radius is None else radius
    if inv_w is None:
        host = nat.to_host(poses_w)
        inv_w = nat.to_dev(np.stack([RigidTransform(r[:9].reshape(3, 3), r[9:]).inverse().as_row12()
                                     for r in host]), np.float64)
    if updated is None:
        updated = nat.zeros((1,), np.int64)
    cmin, cmax = float(np.float32(clip_min)), float(np.float32(clip_max))
    math = lm.default_math()

    frames = frames.contiguous()
    poses_w = poses_w.contiguous()
    inv_w = inv_w.contiguous()

    def issue():
        # activation of frame f+1 overlaps the integration of frame f
        nat.call("rk_grid_integrate_frames", h, sensor, nat.ptr(frames), int(frames.shape[0]),
                 nat.ptr(poses_w), nat.ptr(inv_w), float(radius), cmin, cmax, math,
                 nat.ptr(updated), nat.stream_ptr())

    if not graph:
        issue()
    else:
        # graphs live on the grid (dropped when its tables are reallocated)
        key = (sensor, frames.data_ptr(), tuple(frames.shape), poses_w.data_ptr(),
               inv_w.data_ptr(), updated.data_ptr(), float(radius), cmin, cmax, math)
        g = grid._graphs.get(key)
        if g is None:
            torch = nat.torch()
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(g, stream=side):
                issue()
            torch.cuda.current_stream().wait_stream(side)
            grid._graphs[key] = g
        g.replay()
    grid.blocks._bump()
    return updated


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
