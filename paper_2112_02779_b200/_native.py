"""ctypes binding of librkb200.so (include/rkb200.h) -- the package's only path
to compute.  There is deliberately no fallback: if the library or a GPU is
missing, every compute entry point raises ``DeviceError``.

PyTorch is used only as plumbing: device allocation, the current CUDA stream
and host<->device copies.  Kernel arguments are raw ``data_ptr()`` values.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import STATUS_TO_ERROR, DeviceError

LIB_PATH = Path(os.environ.get("RK_LIB") or Path(__file__).resolve().parent / "lib" / "librkb200.so")

_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_f32 = C.c_float
_f64 = C.c_double


class SensorDesc(C.Structure):
    _fields_ = [("height", _i32), ("width", _i32), ("receiver_radius", _f64),
                ("dirs_host", _p), ("origins_host", _p), ("azimuth_host", _p),
                ("elevation_host", _p), ("inv_rows_host", _p), ("inv_size", _i32),
                ("inv_phi_min", _f64), ("inv_phi_max", _f64),
                ("fov_lo", _f64), ("fov_hi", _f64)]


class IcpConfig(C.Structure):
    _fields_ = [("kernel_scale", _f64), ("max_dist", _f64), ("rot_eps", _f64),
                ("trans_eps", _f64), ("clip_min", _f32), ("clip_max", _f32),
                ("n_levels", _i32), ("strides", _i32 * 8), ("iters", _i32 * 8),
                ("min_corr", _i32), ("scale_with_stride", _i32), ("math", _i32),
                ("surfel_pitch", _i64), ("surfel_level_off", _i32 * 8),
                ("n_src_images", _i32), ("n_dst_images", _i32)]


# name -> argtypes (restype is always int status)
SIGNATURES = {
    "rk_last_error": [C.c_char_p, C.c_size_t],
    "rk_version": [],
    "rk_struct_size": [C.c_int],
    "rk_sensor_create": [C.POINTER(SensorDesc), C.POINTER(_p)],
    "rk_sensor_destroy": [_p],
    "rk_project_f32": [_p, _p, _i64, C.c_int, _p, _p, _p, _p, _p],
    "rk_svml_eval": [_p, C.c_int, _p, _p, _i64, _p, _p],
    "rk_project_f64": [_p, _p, _i64, C.c_int, _f64, C.c_int, _p, _p, _p, _p, _p, _p],
    "rk_row_from_elevation": [_p, _p, C.c_int, _i64, _p, _p],
    "rk_inverse_lut_lookup": [_p, _i32, _f64, _f64, _p, C.c_int, _i64, _p, _p],
    "rk_unproject_many": [_p, _p, _p, _p, _i64, _p, _p],
    "rk_unproject_image": [_p, _p, _i32, _p, _p],
    "rk_normals_cross": [_p, _p, _i32, _p, _p, _p, _p],
    "rk_stride_compact": [_p, _p, _i32, _i32, _f32, _f32, _p, _p, _p],
    "rk_normals_cross_pyramid": [_p, _p, _i32, _p, _i32, _p, _i64, _p],
    "rk_surfel_record_floats": [],
    "rk_normals_pca": [_p, _p, _i32, _i32, _f64, _f64, _p, _p, _p, _p],
    "rk_zbuffer_image": [_p, _p, _p, _p, _p, _i64, _p, _p, _p, _p],
    "rk_unproject_pixels": [_p, _p, _p, _p, _i64, _p, _p],
    "rk_compact_mask": [_p, _i64, _p, _p, _p],
    "rk_correspondences_f32": [_p, _p, _i64, _p, _p, _p, _f64, _i32, C.c_int, _p, _p, _p, _p],
    "rk_make_surfel": [_p, _p, _p, _i64, _p, _p],
    "rk_register_batch": [_p, _p, _p, _p, _p, _p, _i32, _p, C.POINTER(IcpConfig), _p, _p, _p,
                          _p, _i32, _p, _p],
    "rk_icp_cluster_capacity": [C.c_int, C.c_int],
    "rk_transform_points": [_p, _p, _i64, _p, _p],
    "rk_associate_f64": [_p, _p, _p, _p, _p, _i64, _p, _f64, _i32, _p, _p, _p, _p],
    "rk_normal_equations_f64": [_p, _p, _p, _p, _i64, _f64, _p, _p, _p],
    "rk_point_to_plane_residuals": [_p, _p, _p, _p, _i64, _p, _p],
    "rk_centroid_translation": [_p, _i64, _p, _i64, _p, _p, _p],
    "rk_grid_create": [_f64, _f64, _f32, _i32, _i64, C.POINTER(_p)],
    "rk_grid_destroy": [_p],
    "rk_grid_reserve": [_p, _i64, _p],
    "rk_grid_clear": [_p, _p],
    "rk_grid_set_shard": [_p, _i32, _i32],
    "rk_block_owner": [_p, _i64, _i32, _p],
    "rk_grid_touch_stats": [_p, _p, _p],
    "rk_grid_set_global_touch": [_p, _p],
    "rk_grid_info": [_p, _p, _p],
    "rk_grid_activate_points": [_p, _p, _i64, _f64, _p],
    "rk_grid_activate_image": [_p, _p, _p, _p, _f64, _f32, _f32, _p],
    "rk_grid_set_touched": [_p, _p, _i64, _p],
    "rk_grid_integrate": [_p, _p, _p, _p, _f32, _f32, C.c_int, _p, _p],
    "rk_grid_integrate_frames": [_p, _p, _p, _i32, _p, _p, _f64, _f32, _f32, C.c_int, _p, _p],
    "rk_grid_reserve_slots": [_p, _i32, _p],
    "rk_grid_activate_frames": [_p, _p, _p, _i32, _p, _f64, _f32, _f32, _p],
    "rk_grid_touch_stats_frames": [_p, _i32, _p, _p],
    "rk_grid_integrate_activated": [_p, _p, _p, _i32, _p, _p, _f32, _f32, C.c_int, _p, _p],
    "rk_grid_keys": [_p, C.c_int, _p, _i64, _p, _p],
    "rk_grid_read_blocks": [_p, _p, _i64, _p, _p, _p],
    "rk_grid_write_blocks": [_p, _p, _i64, _p, _p],
    "rk_grid_query": [_p, _p, _i64, _p, _p, _p, _p],
    "rk_render": [_p, _p, _i32, _p, _i32, _p, _p],
    "rk_mc_extract": [_p, _p, _f32, C.POINTER(_p), _p],
    "rk_mesh_info": [_p, _p],
    "rk_mesh_copy": [_p, _p, _p, _p, _p],
    "rk_mesh_free": [_p],
}

_lib = None


def load(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load (once) and type the shared library; raise DeviceError if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise DeviceError(f"librkb200.so not built ({p}); run __graft_entry__.build()")
    lib = C.CDLL(str(p))
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    for which, st in ((0, SensorDesc), (1, IcpConfig)):
        if lib.rk_struct_size(which) != C.sizeof(st):
            raise DeviceError(f"{p.name}: {st.__name__} is {C.sizeof(st)} bytes here, "
                              f"{lib.rk_struct_size(which)} in the library (stale build?)")
    if path is None:
        _lib = lib
    return lib


def last_error() -> str:
    buf = C.create_string_buffer(512)
    load().rk_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    cls = STATUS_TO_ERROR.get(int(status), DeviceError)
    msg = last_error() or what
    raise cls(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


# ------------------------------------------------------------------ torch plumbing

def torch():
    import torch as _t
    return _t


def device():
    t = torch()
    if not t.cuda.is_available():
        raise DeviceError("no CUDA device visible: this package has no CPU path")
    return t.device("cuda", t.cuda.current_device())


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


def ptr(x) -> int | None:
    return None if x is None else x.data_ptr()


_NP2T = {np.dtype(np.float32): "float32", np.dtype(np.float64): "float64",
         np.dtype(np.int32): "int32", np.dtype(np.int64): "int64",
         np.dtype(np.uint8): "uint8", np.dtype(np.int8): "int8", np.dtype(bool): "bool"}


def to_dev(a, dtype) -> "object":
    """numpy / torch input -> contiguous CUDA tensor of numpy ``dtype``."""
    t = torch()
    tdt = getattr(t, _NP2T[np.dtype(dtype)])
    if isinstance(a, t.Tensor):
        return a.to(device=device(), dtype=tdt).contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=dtype))
    return t.from_numpy(arr).to(device(), non_blocking=False)


def empty(shape, dtype):
    t = torch()
    return t.empty(shape, dtype=getattr(t, _NP2T[np.dtype(dtype)]), device=device())


def zeros(shape, dtype):
    t = torch()
    return t.zeros(shape, dtype=getattr(t, _NP2T[np.dtype(dtype)]), device=device())


def to_host(x) -> np.ndarray:
    return x.detach().cpu().numpy()


def is_tensor(x) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, _t.Tensor)
