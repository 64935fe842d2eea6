"""Cylindrical spinning-LiDAR sensor model -- drop-in for rangekit/lidar_model.py.

Host side: ``LidarIntrinsics`` validates the calibration and derives the ray
tables with the reference's own numpy expressions (lidar_model.py:128-179), so
the float64 tables the kernels read are bit-identical to the reference's.
They are uploaded once per device (``device_sensor``).

Device side: ``project_many`` / ``row_from_elevation`` / ``unproject_many`` /
``InverseElevationLut.lookup`` run in librkb200.so.  Inputs may be numpy arrays
(results come back as numpy, like the reference) or CUDA tensors (results stay
on the device).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np

from . import _native as nat
from .errors import DegenerateRange, InvalidIntrinsics, OutOfFov

TWO_PI = 2.0 * np.pi

MODE_CALIBRATED = "calibrated"
MODE_SYNTHETIC = "synthetic"

PROJ_OK = 0
PROJ_OUT_OF_FOV = 1
PROJ_DEGENERATE = 2

MATH_FAST = 0   # minimax atan2 / asin (<= 2.5 ulp) + MUFU square roots, float32 ICP move
MATH_CR = 1     # float64-evaluated, rounded once (parity mode)
MATH_LIBM = 2   # CUDA atan2f / asinf (<= 2 ulp), IEEE division (project_many only)
MATH_NP = 3     # numpy's own float32 arctan2 / arcsin (SVML, rk_svml.cuh), float64 ICP move:
                # the reference's projection bit for bit (default)

_default_math = MATH_NP


def set_default_math(mode: int) -> None:
    """Select the projection arithmetic of every bulk kernel: MATH_NP (default,
    the reference's own bits), MATH_FAST (faster, within the tolerance
    contract), MATH_CR (correctly rounded transcendentals)."""
    global _default_math
    if int(mode) not in (MATH_FAST, MATH_CR, MATH_LIBM, MATH_NP):
        raise ValueError(f"unknown math mode {mode}")
    _default_math = int(mode)


def default_math() -> int:
    return _default_math


class math_mode:
    """``with math_mode(MATH_FAST): ...`` -- the default mode inside the block,
    restored on exit."""

    def __init__(self, mode: int):
        self.mode = int(mode)

    def __enter__(self):
        self.prev = default_math()
        set_default_math(self.mode)
        return self

    def __exit__(self, *exc):
        set_default_math(self.prev)
        return False


def round_half_up(x):
    """floor(x + 0.5) as int64 (lidar_model.py:36-38)."""
    return np.floor(np.asarray(x) + 0.5).astype(np.int64)


@dataclass(frozen=True)
class InverseElevationLut:
    """Uniform elevation bins -> nearest row (lidar_model.py:48-66)."""

    rows: np.ndarray
    phi_min: float
    phi_max: float

    @property
    def size(self) -> int:
        return self.rows.shape[0]

    def lookup(self, phi):
        """Nearest-bin row estimate on the device; float32 phi stays float32."""
        back = not nat.is_tensor(phi)
        ph = phi if not back else np.asarray(phi)
        is64 = (str(ph.dtype) in ("float64", "torch.float64"))
        d_phi = nat.to_dev(ph, np.float64 if is64 else np.float32)
        shape = tuple(d_phi.shape)
        rows = nat.to_dev(self.rows, np.int32)
        out = nat.empty(shape, np.int32)
        nat.call("rk_inverse_lut_lookup", nat.ptr(rows), self.size, float(self.phi_min),
                 float(self.phi_max), nat.ptr(d_phi), int(is64), d_phi.numel(), nat.ptr(out),
                 nat.stream_ptr())
        return nat.to_host(out) if back else out


def build_inverse_elevation_lut(elevation_lut, factor: int = 2) -> InverseElevationLut:
    """factor*H bins over the LUT span, nearest row per bin, lowest row on ties
    (lidar_model.py:69-91).  Host-side table construction (once per sensor)."""
    el = np.asarray(elevation_lut, dtype=float)
    H = el.shape[0]
    if H < 2:
        raise InvalidIntrinsics("elevation LUT needs at least 2 rows")
    if factor < 2:
        raise InvalidIntrinsics("inverse LUT factor must be >= 2")
    steps = np.diff(el)
    if not (np.all(steps > 0) or np.all(steps < 0)):
        raise InvalidIntrinsics("elevation LUT must be strictly monotonic")
    lo, hi = float(el.min()), float(el.max())
    centres = np.linspace(lo, hi, factor * H)
    rows = np.argmin(np.abs(el[None, :] - centres[:, None]), axis=1)
    return InverseElevationLut(rows.astype(np.int32), lo, hi)


@dataclass(frozen=True)
class LidarIntrinsics:
    """Immutable sensor description (lidar_model.py:94-202)."""

    width: int
    height: int
    receiver_radius: float
    azimuth_lut: np.ndarray
    elevation_lut: np.ndarray
    mode: str = MODE_CALIBRATED
    inv_factor: int = 2

    def __post_init__(self):
        az = np.asarray(self.azimuth_lut, dtype=float).reshape(-1)
        el = np.asarray(self.elevation_lut, dtype=float).reshape(-1)
        object.__setattr__(self, "azimuth_lut", az)
        object.__setattr__(self, "elevation_lut", el)
        if self.width < 2 or self.height < 2:
            raise InvalidIntrinsics("width and height must be >= 2")
        if az.shape[0] != self.height or el.shape[0] != self.height:
            raise InvalidIntrinsics("LUT lengths must equal the image height")
        if self.receiver_radius < 0:
            raise InvalidIntrinsics("receiver radius must be >= 0")
        if np.any(np.abs(az) >= np.pi):
            raise InvalidIntrinsics("azimuth offsets must lie in (-pi, pi)")
        if self.mode not in (MODE_CALIBRATED, MODE_SYNTHETIC):
            raise InvalidIntrinsics(f"unknown mode {self.mode!r}")
        if self.mode == MODE_SYNTHETIC and (self.receiver_radius != 0.0 or np.any(az != 0.0)):
            raise InvalidIntrinsics("synthetic mode requires r0 = 0 and zero azimuth offsets")
        object.__setattr__(self, "inv_elevation_lut",
                           build_inverse_elevation_lut(el, self.inv_factor))

    inv_elevation_lut: InverseElevationLut = field(init=False, repr=False)

    def __hash__(self):
        return id(self)

    def __eq__(self, other):
        return self is other

    @cached_property
    def fov_bounds(self) -> tuple[float, float]:
        el = self.elevation_lut
        H = el.shape[0]
        lo_end = 0 if el[0] < el[-1] else H - 1
        hi_end = H - 1 - lo_end
        gap_lo = abs(el[lo_end] - el[lo_end - 1 if lo_end else 1])
        gap_hi = abs(el[hi_end] - el[hi_end - 1 if hi_end else 1])
        return float(el.min() - 0.5 * gap_lo), float(el.max() + 0.5 * gap_hi)

    @cached_property
    def ray_dirs(self) -> np.ndarray:
        """(H, W, 3) unit ray directions (same numpy expressions as the reference)."""
        col_angle = TWO_PI * np.arange(self.width) / self.width
        theta = col_angle[None, :] + self.azimuth_lut[:, None]
        cphi = np.cos(self.elevation_lut[:, None])
        return np.stack([np.cos(theta) * cphi,
                         np.sin(theta) * cphi,
                         np.broadcast_to(np.sin(self.elevation_lut[:, None]), theta.shape)], axis=-1)

    @cached_property
    def ray_origins(self) -> np.ndarray:
        col_angle = TWO_PI * np.arange(self.width) / self.width
        return np.stack([self.receiver_radius * np.cos(col_angle),
                         self.receiver_radius * np.sin(col_angle),
                         np.zeros(self.width)], axis=-1)

    @cached_property
    def ray_tables_flat(self):
        dirs = tuple(np.ascontiguousarray(self.ray_dirs[..., c].reshape(-1)) for c in range(3))
        origins = tuple(np.ascontiguousarray(self.ray_origins[:, c]) for c in range(3))
        return dirs, origins

    @cached_property
    def ray_tables_flat_f32(self):
        dirs, origins = self.ray_tables_flat
        return tuple(d.astype(np.float32) for d in dirs), tuple(o.astype(np.float32) for o in origins)

    @cached_property
    def _luts_f32(self):
        return self.azimuth_lut.astype(np.float32), self.elevation_lut.astype(np.float32)

    def row_from_elevation(self, phi):
        """Row minimising |elevation_lut[v] - phi| (inverse LUT + ±1 refine) on
        the device; float32 input runs the float32 path."""
        back = not nat.is_tensor(phi)
        ph = np.asarray(phi) if back else phi
        is64 = str(ph.dtype) in ("float64", "torch.float64")
        d_phi = nat.to_dev(ph, np.float64 if is64 else np.float32)
        out = nat.empty(tuple(d_phi.shape), np.int32)
        nat.call("rk_row_from_elevation", device_sensor(self), nat.ptr(d_phi), int(is64),
                 d_phi.numel(), nat.ptr(out), nat.stream_ptr())
        return nat.to_host(out) if back else out


# ------------------------------------------------------------------ device sensor

class _DeviceSensor:
    def __init__(self, intr: LidarIntrinsics):
        lib = nat.load()
        dirs = np.ascontiguousarray(intr.ray_dirs.reshape(-1), dtype=np.float64)
        orig = np.ascontiguousarray(intr.ray_origins.reshape(-1), dtype=np.float64)
        az = np.ascontiguousarray(intr.azimuth_lut, dtype=np.float64)
        el = np.ascontiguousarray(intr.elevation_lut, dtype=np.float64)
        inv = intr.inv_elevation_lut
        rows = np.ascontiguousarray(inv.rows, dtype=np.int32)
        lo, hi = intr.fov_bounds
        desc = nat.SensorDesc(intr.height, intr.width, float(intr.receiver_radius),
                              dirs.ctypes.data, orig.ctypes.data, az.ctypes.data, el.ctypes.data,
                              rows.ctypes.data, rows.shape[0], float(inv.phi_min),
                              float(inv.phi_max), float(lo), float(hi))
        handle = C.c_void_p()
        nat.check(lib.rk_sensor_create(C.byref(desc), C.byref(handle)), "rk_sensor_create")
        self.handle = handle.value
        self._lib = lib

    def __del__(self):
        try:
            self._lib.rk_sensor_destroy(self.handle)
        except Exception:
            pass


def device_sensor(intr: LidarIntrinsics) -> int:
    """Opaque ``rk_sensor*`` for intr on the current device (cached)."""
    dev = nat.device()
    cache = intr.__dict__.setdefault("_device_sensors", {})
    s = cache.get(dev.index)
    if s is None:
        s = cache[dev.index] = _DeviceSensor(intr)
    return s.handle


def synthetic_intrinsics(height: int, width: int, fov_min: float, fov_max: float) -> LidarIntrinsics:
    """Uniform bin-centre elevations, row 0 at the top (lidar_model.py:205-224)."""
    if not fov_min < fov_max:
        raise InvalidIntrinsics("fov_min must be < fov_max")
    if height < 2 or width < 2:
        raise InvalidIntrinsics("width and height must be >= 2")
    v = np.arange(height)
    elev = fov_max - (v + 0.5) * (fov_max - fov_min) / height
    return LidarIntrinsics(width=width, height=height, receiver_radius=0.0,
                           azimuth_lut=np.zeros(height), elevation_lut=elev, mode=MODE_SYNTHETIC)


@dataclass(frozen=True)
class PixelRay:
    u: float
    v: int
    r: float


def unproject_many(u, v, r, intr: LidarIntrinsics):
    """(u, v, r) -> (..., 3) sensor-frame points (lidar_model.py:236-250)."""
    back = not nat.is_tensor(u)
    du = nat.to_dev(u, np.float64)
    shape = tuple(du.shape)
    dv = nat.to_dev(np.broadcast_to(np.asarray(v) if back else v.cpu().numpy(), shape) if back
                    else v.expand(shape), np.int64)
    dr = nat.to_dev(np.broadcast_to(np.asarray(r, dtype=float), shape) if back
                    else r.expand(shape), np.float64)
    out = nat.empty(shape + (3,), np.float64)
    nat.call("rk_unproject_many", device_sensor(intr), nat.ptr(du), nat.ptr(dv), nat.ptr(dr),
             du.numel(), nat.ptr(out), nat.stream_ptr())
    return nat.to_host(out) if back else out


def unproject(u: float, v: int, r: float, intr: LidarIntrinsics):
    if not (0 <= u < intr.width and 0 <= v < intr.height):
        raise ValueError(f"pixel ({u}, {v}) outside {intr.height}x{intr.width} grid")
    if not (np.isfinite(r) and r >= 0):
        raise ValueError("range must be finite and >= 0")
    return unproject_many(u, v, r, intr)


def project_many(points, intr: LidarIntrinsics, max_iters: int = 3, tol: float = 1e-4,
                 single: bool = False, refine: bool = True, math: int | None = None):
    """Vectorised projection -> (u, v, r, status) (lidar_model.py:262-344).

    single=True is the bulk float32 path (closed-form receiver, no refine);
    single=False the float64 fixed-point path with optional refine pass.
    """
    back = not nat.is_tensor(points)
    dt = np.float32 if single else np.float64
    pts = nat.to_dev(points, dt)
    shape = tuple(pts.shape[:-1])
    n = int(np.prod(shape)) if shape else 1
    u = nat.empty(shape, dt)
    v = nat.empty(shape, np.int32)
    r = nat.empty(shape, dt)
    st = nat.empty(shape, np.int8)
    sensor = device_sensor(intr)
    if single:
        nat.call("rk_project_f32", sensor, nat.ptr(pts), n, _default_math if math is None else math,
                 nat.ptr(u), nat.ptr(v), nat.ptr(r), nat.ptr(st), nat.stream_ptr())
    else:
        work = nat.empty((3 * n + 4,), np.float64)
        nat.call("rk_project_f64", sensor, nat.ptr(pts), n, int(max_iters), float(tol),
                 int(bool(refine)), nat.ptr(u), nat.ptr(v), nat.ptr(r), nat.ptr(st),
                 nat.ptr(work), nat.stream_ptr())
    if back:
        vv = nat.to_host(v)
        return nat.to_host(u), (vv if single else vv.astype(np.int64)), nat.to_host(r), nat.to_host(st)
    return u, v, r, st


def project(p, intr: LidarIntrinsics, max_iters: int = 3, tol: float = 1e-4) -> PixelRay:
    """One point; raises OutOfFov / DegenerateRange (lidar_model.py:347-357)."""
    u, v, r, status = project_many(np.asarray(p, dtype=float).reshape(1, 3), intr,
                                   max_iters=max_iters, tol=tol)
    code = int(status[0])
    if code == PROJ_DEGENERATE:
        raise DegenerateRange("point lies on or inside the receiver cylinder")
    if code == PROJ_OUT_OF_FOV:
        raise OutOfFov("point elevation outside the sensor field of view")
    return PixelRay(u=float(u[0]), v=int(v[0]), r=float(r[0]))
