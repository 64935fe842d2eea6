"""Zero-crossing mesh extraction on the device -- drop-in for
rangekit/mesh_extract.py (K6 ``rk_mc_extract``)."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .trace import nvtx
from .mc_tables import TRI_TABLE
from .sdf_volume import VoxelBlockGrid


@dataclass
class TriangleMesh:
    vertices: np.ndarray
    triangles: np.ndarray
    normals: np.ndarray | None = None

    def __post_init__(self):
        self.vertices = np.asarray(self.vertices, dtype=float).reshape(-1, 3)
        self.triangles = np.asarray(self.triangles, dtype=np.int32).reshape(-1, 3)
        if self.normals is not None:
            self.normals = np.asarray(self.normals, dtype=float).reshape(-1, 3)

    @property
    def n_vertices(self) -> int:
        return self.vertices.shape[0]

    @property
    def n_triangles(self) -> int:
        return self.triangles.shape[0]


_table_cache = {}


def _device_table():
    dev = nat.device()
    t = _table_cache.get(dev.index)
    if t is None:
        t = _table_cache[dev.index] = nat.to_dev(TRI_TABLE, np.int8)
    return t


def extract_mesh_device(grid: VoxelBlockGrid, min_weight: float = 1.0):
    """Marching Cubes -> (vertices (V,3) f64, triangles (T,3) i32, normals (V,3) f64)
    as CUDA tensors."""
    h = grid._prepare()
    lib = nat.load()
    mesh = C.c_void_p()
    nat.check(lib.rk_mc_extract(h, nat.ptr(_device_table()), float(np.float32(min_weight)),
                                C.byref(mesh), nat.stream_ptr()), "rk_mc_extract")
    try:
        counts = np.zeros(2, np.int64)
        nat.check(lib.rk_mesh_info(mesh, counts.ctypes.data), "rk_mesh_info")
        nv, nt = int(counts[0]), int(counts[1])
        v = nat.empty((nv, 3), np.float64)
        n = nat.empty((nv, 3), np.float64)
        t = nat.empty((nt, 3), np.int32)
        nat.check(lib.rk_mesh_copy(mesh, nat.ptr(v), nat.ptr(n), nat.ptr(t), nat.stream_ptr()),
                  "rk_mesh_copy")
        nat.torch().cuda.current_stream().synchronize()
    finally:
        lib.rk_mesh_free(mesh)
    return v, t, n


@nvtx("extract_mesh")
def extract_mesh(grid: VoxelBlockGrid, min_weight: float = 1.0) -> TriangleMesh:
    """Marching Cubes over every cell whose 8 corners have weight >= min_weight
    (mesh_extract.py:85-178)."""
    v, t, n = extract_mesh_device(grid, min_weight)
    return TriangleMesh(nat.to_host(v), nat.to_host(t), nat.to_host(n))
