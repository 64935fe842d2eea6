"""Globally sparse, locally dense TSDF on the device -- drop-in for
rangekit/sdf_volume.py.

``VoxelBlockGrid`` owns an ``rk_grid`` (device voxel-block pool + hash).  Its
``blocks`` attribute is a lazy mapping that materialises ``VoxelBlock`` host
copies on access and writes back host-side edits before the next device
operation, so code written against the reference's ``dict`` (including tests
that fill blocks by hand or read ``grid.blocks[key].tsdf``) keeps working.
"""

from __future__ import annotations

import ctypes as C
from collections.abc import MutableMapping
from dataclasses import dataclass, field
from itertools import product

import numpy as np

from . import _native as nat
from .trace import nvtx
from . import lidar_model as lm
from .errors import DeviceError, InvalidPose
from .range_image import RangeImage
from .se3 import RigidTransform

BLOCK_EDGE = 16
BLOCK_VOXELS = BLOCK_EDGE ** 3
_LOCAL_OFFSETS = np.array(list(product(range(BLOCK_EDGE), repeat=3)), dtype=np.int64)
_INITIAL_CAPACITY = 1024


class VoxelBlock:
    """16^3 {tsdf, weight} float32 arrays (sdf_volume.py:29-32).  Blocks handed
    out by a grid refresh themselves from the device after device updates."""

    def __init__(self, tsdf=None, weight=None):
        self._tsdf = np.zeros((BLOCK_EDGE,) * 3, np.float32) if tsdf is None else tsdf
        self._weight = np.zeros((BLOCK_EDGE,) * 3, np.float32) if weight is None else weight
        self._owner = None
        self._key = None
        self._ver = -1

    def _sync(self):
        o = self._owner
        if o is not None and self._ver != o._version:
            o._refresh([self._key])

    @property
    def tsdf(self):
        self._sync()
        return self._tsdf

    @tsdf.setter
    def tsdf(self, value):
        self._sync()
        self._tsdf = value
        if self._owner is not None:
            self._owner._dirty.add(self._key)

    @property
    def weight(self):
        self._sync()
        return self._weight

    @weight.setter
    def weight(self, value):
        self._sync()
        self._weight = value
        if self._owner is not None:
            self._owner._dirty.add(self._key)


class _DeviceBlocks(MutableMapping):
    """dict-like view of the device pool keyed by (i, j, k)."""

    def __init__(self, grid: "VoxelBlockGrid"):
        self._grid = grid
        self._objs: dict[tuple, VoxelBlock] = {}
        self._dirty: set[tuple] = set()   # host objects that may differ from the device
        self._version = 0
        self._keys_cache = None

    # -- device bookkeeping
    def _bump(self):
        self._version += 1
        self._keys_cache = None

    def _device_keys(self):
        if self._keys_cache is None:
            g = self._grid
            if g._handle is None:
                self._keys_cache = []
            else:
                self._keys_cache = [tuple(k) for k in g._export_keys(touched=False).tolist()]
        return self._keys_cache

    def _refresh(self, keys):
        """Fetch device values of keys into their host objects."""
        g = self._grid
        keys = [k for k in keys if k not in self._dirty]
        if not keys or g._handle is None:
            return
        kd = nat.to_dev(np.asarray(keys, dtype=np.int32).reshape(-1, 3), np.int32)
        vox = nat.empty((len(keys), BLOCK_VOXELS, 2), np.float32)
        found = nat.empty((len(keys),), np.uint8)
        nat.call("rk_grid_read_blocks", g._handle, nat.ptr(kd), len(keys), nat.ptr(vox),
                 nat.ptr(found), nat.stream_ptr())
        host = nat.to_host(vox)
        for j, k in enumerate(keys):
            obj = self._objs[k]
            obj._tsdf = np.ascontiguousarray(host[j, :, 0]).reshape((BLOCK_EDGE,) * 3)
            obj._weight = np.ascontiguousarray(host[j, :, 1]).reshape((BLOCK_EDGE,) * 3)
            obj._ver = self._version
            # handed-out arrays may be edited in place: write them back before
            # the next device operation
            self._dirty.add(k)

    def flush(self):
        """Upload host-side edits (and hand-inserted blocks) to the device."""
        if not self._dirty:
            return
        g = self._grid
        keys = sorted(self._dirty)
        vox = np.empty((len(keys), BLOCK_VOXELS, 2), np.float32)
        for j, k in enumerate(keys):
            o = self._objs[k]
            vox[j, :, 0] = np.asarray(o._tsdf, dtype=np.float32).reshape(-1)
            vox[j, :, 1] = np.asarray(o._weight, dtype=np.float32).reshape(-1)
        g._ensure()
        g._ensure_capacity(len(self) + len(keys))
        kd = nat.to_dev(np.asarray(keys, dtype=np.int32).reshape(-1, 3), np.int32)
        vd = nat.to_dev(vox, np.float32)
        nat.call("rk_grid_write_blocks", g._handle, nat.ptr(kd), len(keys), nat.ptr(vd),
                 nat.stream_ptr())
        self._dirty.clear()
        self._keys_cache = None
        for k in keys:
            self._objs[k]._ver = self._version

    # -- mapping protocol
    def __getitem__(self, key):
        key = tuple(int(x) for x in key)
        obj = self._objs.get(key)
        if obj is not None:
            return obj
        if key not in set(self._device_keys()):
            raise KeyError(key)
        obj = VoxelBlock()
        obj._owner, obj._key, obj._ver = self, key, -1
        self._objs[key] = obj
        self._refresh([key])
        return obj

    def __setitem__(self, key, blk):
        key = tuple(int(x) for x in key)
        if not isinstance(blk, VoxelBlock):
            raise TypeError("blocks values must be VoxelBlock")
        blk._owner, blk._key, blk._ver = self, key, self._version
        self._objs[key] = blk
        self._dirty.add(key)

    def __delitem__(self, key):
        raise TypeError("voxel blocks are never removed (sdf_volume.py: blocks only grow)")

    def _all_keys(self):
        dk = self._device_keys()
        extra = [k for k in self._dirty if k not in set(dk)]
        return dk + sorted(extra)

    def __iter__(self):
        return iter(self._all_keys())

    def __len__(self):
        return len(self._all_keys())

    def __contains__(self, key):
        key = tuple(int(x) for x in key)
        return key in self._objs or key in set(self._device_keys())

    def items(self):
        keys = self._all_keys()
        missing = [k for k in keys if k not in self._objs]
        for k in missing:
            obj = VoxelBlock()
            obj._owner, obj._key, obj._ver = self, k, -1
            self._objs[k] = obj
        stale = [k for k in keys if self._objs[k]._ver != self._version]
        self._refresh(stale)
        return [(k, self._objs[k]) for k in keys]

    def values(self):
        return [v for _, v in self.items()]


@dataclass
class VoxelBlockGrid:
    """Sparse 16^3-block TSDF (sdf_volume.py:35-61), stored on the device."""

    voxel_size: float
    truncation: float | None = None
    max_weight: float = 100.0
    integrate_free_space: bool = True
    capacity: int = _INITIAL_CAPACITY
    blocks: _DeviceBlocks = field(init=False, repr=False)

    def __post_init__(self):
        if self.voxel_size <= 0:
            raise ValueError("voxel size must be > 0")
        if self.truncation is None:
            self.truncation = 4.0 * self.voxel_size
        if self.truncation <= 0:
            raise ValueError("truncation must be > 0")
        self._handle = None
        self._lib = None
        self._graphs = {}   # CUDA graphs recorded against this grid's tables (pipeline.py)
        self.blocks = _DeviceBlocks(self)

    # -- device handle
    def _ensure(self):
        if self._handle is None:
            lib = nat.load()
            h = C.c_void_p()
            nat.check(lib.rk_grid_create(float(self.voxel_size), float(self.truncation),
                                         float(np.float32(self.max_weight)),
                                         int(bool(self.integrate_free_space)), int(self.capacity),
                                         C.byref(h)), "rk_grid_create")
            self._handle = h.value
            self._lib = lib
        return self._handle

    def __del__(self):
        if getattr(self, "_handle", None) is not None:
            try:
                self._lib.rk_grid_destroy(self._handle)
            except Exception:
                pass

    MAX_GRAPHS = 32

    def cache_graph(self, key, entry):
        """Keep a recorded CUDA graph (bounded: the oldest entry is dropped
        beyond MAX_GRAPHS, so callers passing fresh buffers cannot grow the
        cache without limit)."""
        while len(self._graphs) >= self.MAX_GRAPHS:
            self._graphs.pop(next(iter(self._graphs)))
        self._graphs[key] = entry

    def check_overflow(self):
        """Raise if an activation ran out of pool capacity (new blocks got no
        slot and were skipped) -- synchronises."""
        n_blocks, cap, overflow, _ = self.info()
        if overflow:
            raise DeviceError(f"voxel-block pool overflow: {n_blocks} blocks in a pool of {cap}; "
                              f"call grid.reserve() with a larger capacity before integrating")

    def info(self):
        """(n_blocks, capacity, overflowed, n_touched) -- synchronises."""
        out = np.zeros(4, np.int64)
        nat.call("rk_grid_info", self._ensure(), out.ctypes.data, nat.stream_ptr())
        return tuple(int(x) for x in out)

    def reserve(self, capacity: int):
        """Grow the device pool to at least ``capacity`` blocks."""
        self._ensure()
        if capacity > self.capacity:
            nat.call("rk_grid_reserve", self._handle, int(capacity), nat.stream_ptr())
            self.capacity = int(capacity)
            self._graphs.clear()   # recorded launches point at the old tables
            self.blocks._bump()

    def _ensure_capacity(self, n):
        if n > self.capacity:
            self.reserve(max(n, 2 * self.capacity))

    def _export_keys(self, touched: bool):
        self._ensure()
        n = C.c_int64()
        nat.call("rk_grid_keys", self._handle, int(touched), None, 0, C.byref(n), nat.stream_ptr())
        out = nat.empty((max(n.value, 1), 3), np.int32)
        nat.call("rk_grid_keys", self._handle, int(touched), nat.ptr(out), n.value, C.byref(n),
                 nat.stream_ptr())
        return nat.to_host(out[:n.value])

    def export_blocks(self, device: bool = False):
        """Every stored block in sorted-key order, read back in one device
        call: (keys (n,3) int32, voxels (n,4096,2) float32 {tsdf, weight}) --
        the SDFG snapshot's payload (io_formats.py:267-277).  device=True
        returns CUDA tensors (for collectives) instead of numpy arrays."""
        self._prepare()
        keys = self._export_keys(touched=False)
        if keys.shape[0]:
            keys = keys[np.lexsort((keys[:, 2], keys[:, 1], keys[:, 0]))]
        kd = nat.to_dev(keys.reshape(-1, 3), np.int32)
        vox = nat.empty((keys.shape[0], BLOCK_VOXELS, 2), np.float32)
        if keys.shape[0]:
            nat.call("rk_grid_read_blocks", self._handle, nat.ptr(kd), keys.shape[0], nat.ptr(vox),
                     None, nat.stream_ptr())
        if device:
            return kd, vox
        return keys.reshape(-1, 3), nat.to_host(vox)

    def import_blocks(self, keys, voxels):
        """Insert / overwrite whole blocks in one device call (keys (n,3),
        voxels (n,4096,2) {tsdf, weight}; numpy arrays or CUDA tensors)."""
        n = int(keys.shape[0])
        if n == 0:
            return
        self._prepare()
        self._ensure_capacity(self.info()[0] + n)
        kd = nat.to_dev(keys, np.int32).reshape(n, 3).contiguous()
        vd = nat.to_dev(voxels, np.float32).reshape(n, BLOCK_VOXELS, 2).contiguous()
        nat.call("rk_grid_write_blocks", self._handle, nat.ptr(kd), n, nat.ptr(vd), nat.stream_ptr())
        self.blocks._bump()

    def _prepare(self):
        """Flush host edits; return the device handle."""
        self._ensure()
        self.blocks.flush()
        return self._handle

    # -- reference helpers
    @property
    def block_extent(self) -> float:
        return BLOCK_EDGE * self.voxel_size

    def block(self, key) -> VoxelBlock:
        return self.blocks[key]

    def voxel_centers(self, key) -> np.ndarray:
        base = np.asarray(key, dtype=np.int64) * BLOCK_EDGE
        return (base + _LOCAL_OFFSETS + 0.5) * self.voxel_size


def _retry_on_overflow(grid: VoxelBlockGrid, run):
    """Run an activation; grow the pool and re-run while it overflowed."""
    while True:
        run()
        n_blocks, cap, overflow, _ = grid.info()
        if not overflow:
            grid.blocks._bump()
            return
        grid.reserve(2 * cap)


def activate_blocks(points, grid: VoxelBlockGrid, radius: float) -> set:
    """Insert zeroed blocks meeting each point's cube; return the touched set
    (sdf_volume.py:82-113)."""
    h = grid._prepare()
    pts = nat.to_dev(points, np.float64).reshape(-1, 3)
    n = pts.shape[0]
    if n == 0:
        return set()

    def run():
        nat.call("rk_grid_activate_points", h, nat.ptr(pts), n, float(radius), nat.stream_ptr())

    _retry_on_overflow(grid, run)
    return set(map(tuple, grid._export_keys(touched=True).tolist()))


def _inverse_row12(pose: RigidTransform):
    inv = pose.inverse()  # numpy, exactly like the reference's integrate()
    return nat.to_dev(inv.as_row12(), np.float64)


def integrate(grid: VoxelBlockGrid, img: RangeImage, pose_frame_to_world: RigidTransform,
              frame_keys, clip_min: float = 0.0, clip_max: float = np.inf,
              threads: int | None = None) -> int:
    """Fold one posed image into the given blocks (sdf_volume.py:116-186).
    Returns the number of updated voxels."""
    pose_frame_to_world.validated()
    if img.intrinsics is None:
        raise InvalidPose("range image must carry intrinsics for integration")
    keys = list(frame_keys)
    if not keys:
        return 0
    h = grid._prepare()
    kd = nat.to_dev(np.asarray(keys, dtype=np.int32).reshape(-1, 3), np.int32)
    nat.call("rk_grid_set_touched", h, nat.ptr(kd), len(keys), nat.stream_ptr())
    return _integrate_touched(grid, img, pose_frame_to_world, clip_min, clip_max)


def _integrate_touched(grid, img, pose, clip_min, clip_max, sync=True):
    intr = img.intrinsics
    rng = img.device_data()
    inv = _inverse_row12(pose)
    updated = nat.zeros((1,), np.int64)
    nat.call("rk_grid_integrate", grid._handle, lm.device_sensor(intr), nat.ptr(rng), nat.ptr(inv),
             float(np.float32(clip_min)), float(np.float32(clip_max)), lm.default_math(),
             nat.ptr(updated), nat.stream_ptr())
    grid.blocks._bump()
    return int(updated.item()) if sync else updated


@nvtx("integrate_cloud_frame")
def integrate_cloud_frame(grid: VoxelBlockGrid, img: RangeImage, pose_frame_to_world: RigidTransform,
                          activation_radius: float | None = None, clip_min: float = 0.0,
                          clip_max: float = np.inf, threads: int | None = None) -> int:
    """activate (from the clipped cloud) + integrate, fused on the device
    (sdf_volume.py:198-210)."""
    pose_frame_to_world.validated()
    if img.intrinsics is None:
        raise InvalidPose("range image must carry intrinsics for integration")
    radius = grid.truncation if activation_radius is None else activation_radius
    h = grid._prepare()
    intr = img.intrinsics
    rng = img.device_data()
    pose_d = nat.to_dev(pose_frame_to_world.as_row12(), np.float64)
    sensor = lm.device_sensor(intr)

    def run():
        nat.call("rk_grid_activate_image", h, sensor, nat.ptr(rng), nat.ptr(pose_d),
                 float(radius), float(np.float32(clip_min)), float(np.float32(clip_max)),
                 nat.stream_ptr())

    _retry_on_overflow(grid, run)
    return _integrate_touched(grid, img, pose_frame_to_world, clip_min, clip_max)


def query_sdf_many(grid: VoxelBlockGrid, pts):
    """Trilinear (sdf, weight, observed) over the 8 enclosing voxel centres
    (sdf_volume.py:221-244)."""
    h = grid._prepare()
    p = nat.to_dev(pts, np.float64).reshape(-1, 3)
    n = p.shape[0]
    sdf = nat.empty((n,), np.float64)
    wt = nat.empty((n,), np.float64)
    ok = nat.empty((n,), np.uint8)
    if n:
        nat.call("rk_grid_query", h, nat.ptr(p), n, nat.ptr(sdf), nat.ptr(wt), nat.ptr(ok),
                 nat.stream_ptr())
    return nat.to_host(sdf), nat.to_host(wt), nat.to_host(ok).astype(bool)


def query_sdf(grid: VoxelBlockGrid, x):
    sdf, wt, ok = query_sdf_many(grid, np.asarray(x, dtype=float).reshape(1, 3))
    if not ok[0]:
        return None
    return float(sdf[0]), float(wt[0])
