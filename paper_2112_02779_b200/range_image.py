"""Range images, point clouds, normal maps, stride views -- drop-in for
rangekit/range_image.py.

Containers hold either host numpy data (like the reference; uploaded per call)
or device tensors (results then stay on the device).  All per-pixel work runs
in librkb200.so: K1 ``rk_normals_cross`` (cross normals + the packed surfel map
the ICP kernel gathers) and K2 ``rk_stride_compact`` (row-major survivor
indices of a stride view, bit-identical to ``np.nonzero``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .trace import nvtx
from . import lidar_model as lm
from .errors import InvalidIntrinsics
from .lidar_model import LidarIntrinsics

INVALID_RANGE = 0.0
DISCONTINUITY_ABS = 0.3
DISCONTINUITY_REL = 0.05


def _is_dev(x) -> bool:
    return nat.is_tensor(x) and x.is_cuda


class RangeImage:
    """H x W float32 ranges in metres, 0.0 = no return (range_image.py:25-55).

    ``data`` may be a numpy array (validated and copied to contiguous float32
    like the reference) or a CUDA tensor (kept on the device; ``.data`` then
    materialises a host copy on first access).
    """

    def __init__(self, data, intrinsics: LidarIntrinsics | None = None):
        self.intrinsics = intrinsics
        self._set(data)

    def _set(self, data):
        self._dev = None
        self._host = None
        if _is_dev(data):
            t = nat.torch()
            d = data.detach().to(t.float32).contiguous()
            if d.ndim != 2:
                raise ValueError("range image data must be 2D")
            bad = (~t.isfinite(d)) | (d < 0)
            if bool(bad.any()):
                raise ValueError("ranges must be finite and >= 0")
            self._dev = d
            shape = tuple(d.shape)
        else:
            if nat.is_tensor(data):
                data = data.detach().numpy()
            arr = np.ascontiguousarray(data, dtype=np.float32)
            if arr.ndim != 2:
                raise ValueError("range image data must be 2D")
            if not np.all(np.isfinite(arr)) or np.any(arr < 0):
                raise ValueError("ranges must be finite and >= 0")
            self._host = arr
            shape = arr.shape
        if self.intrinsics is not None and shape != (self.intrinsics.height, self.intrinsics.width):
            raise InvalidIntrinsics("image dimensions do not match intrinsics")

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            self._host = nat.to_host(self._dev)
        return self._host

    @data.setter
    def data(self, value):
        self._set(value)

    @property
    def on_device(self) -> bool:
        return self._dev is not None

    def device_data(self):
        """(H, W) float32 CUDA tensor (uploaded from the host copy if needed)."""
        if self._dev is not None:
            return self._dev
        return nat.to_dev(self._host, np.float32)

    @property
    def height(self) -> int:
        return (self._dev if self._dev is not None else self._host).shape[0]

    @property
    def width(self) -> int:
        return (self._dev if self._dev is not None else self._host).shape[1]

    @property
    def valid_mask(self) -> np.ndarray:
        return self.data > INVALID_RANGE

    def strided(self, stride: int) -> "StridedView":
        return StridedView(self, stride)


class NormalImage:
    """Per-pixel unit normals (range_image.py:58-66): vectors (H,W,3) float32,
    valid (H,W) bool.  Device-born maps also carry the packed ``surfel`` map
    {nx, ny, nz, range-if-valid} the ICP kernel gathers."""

    def __init__(self, vectors, valid, surfel=None):
        self._vec = vectors
        self._valid = valid
        self.surfel = surfel

    @property
    def vectors(self) -> np.ndarray:
        if _is_dev(self._vec):
            self._vec = nat.to_host(self._vec)
        return self._vec

    @vectors.setter
    def vectors(self, v):
        self._vec = v
        self.surfel = None

    @property
    def valid(self) -> np.ndarray:
        if _is_dev(self._valid):
            self._valid = nat.to_host(self._valid).astype(bool)
        return self._valid

    @valid.setter
    def valid(self, v):
        self._valid = v
        self.surfel = None

    def device_surfel(self, img: "RangeImage"):
        """(H, W, 4) float32 device map; built by rk_make_surfel for maps that
        were not produced by the device normal kernel."""
        if self.surfel is not None:
            return self.surfel
        rng = img.device_data()
        vec = nat.to_dev(self._vec, np.float32)
        val = nat.to_dev(self._valid, np.uint8)
        out = nat.empty(tuple(rng.shape) + (4,), np.float32)
        nat.call("rk_make_surfel", nat.ptr(rng), nat.ptr(vec), nat.ptr(val), rng.numel(),
                 nat.ptr(out), nat.stream_ptr())
        return out

    def strided(self, stride: int) -> "StridedView":
        return StridedView(self, stride)


@dataclass(frozen=True)
class StridedView:
    """Zero-copy decimated view: pixel (i, j) reads base pixel (s*i, s*j)
    (range_image.py:69-116).  Pure indexing; the kernels apply the same index
    arithmetic to the level-0 image directly."""

    base: RangeImage | NormalImage
    stride: int

    def __post_init__(self):
        if self.stride < 1:
            raise ValueError("stride must be >= 1")

    def _base_hw(self):
        if isinstance(self.base, RangeImage):
            return self.base.data.shape
        return self.base.valid.shape

    @property
    def shape(self) -> tuple[int, int]:
        h, w = self._base_hw()
        s = self.stride
        return (-(-h // s), -(-w // s))

    @property
    def ranges(self) -> np.ndarray:
        return self.base.data[::self.stride, ::self.stride]

    @property
    def vectors(self) -> np.ndarray:
        return self.base.vectors[::self.stride, ::self.stride]

    @property
    def valid(self) -> np.ndarray:
        if isinstance(self.base, RangeImage):
            return self.base.valid_mask[::self.stride, ::self.stride]
        return self.base.valid[::self.stride, ::self.stride]

    @property
    def base_rows(self) -> np.ndarray:
        return np.arange(0, self._base_hw()[0], self.stride)

    @property
    def base_cols(self) -> np.ndarray:
        return np.arange(0, self._base_hw()[1], self.stride)


@dataclass
class ProjectionStats:
    kept: int = 0
    collisions: int = 0
    out_of_fov: int = 0
    degenerate: int = 0


def _require_intrinsics(img: RangeImage) -> LidarIntrinsics:
    if img.intrinsics is None:
        raise InvalidIntrinsics("range image has no linked intrinsics")
    return img.intrinsics


def _ret(img: RangeImage, t):
    return t if img.on_device else nat.to_host(t)


def unproject_image(img: RangeImage):
    """(H, W, 3) float64 sensor-frame points for every pixel (range_image.py:129-133)."""
    intr = _require_intrinsics(img)
    rng = img.device_data()
    out = nat.empty((intr.height, intr.width, 3), np.float64)
    nat.call("rk_unproject_image", lm.device_sensor(intr), nat.ptr(rng), 1, nat.ptr(out),
             nat.stream_ptr())
    return _ret(img, out)


def stride_indices(img: RangeImage, stride: int, clip_min: float = 0.0, clip_max: float = np.inf):
    """K2: row-major flat base indices (v*W + u) of the stride view's survivors
    (mask r > 0 & clip_min <= r <= clip_max, compared in float32) -> device int32."""
    intr = _require_intrinsics(img)
    rng = img.device_data()
    Hs, Ws = -(-intr.height // stride), -(-intr.width // stride)
    idx = nat.empty((Hs * Ws,), np.int32)
    cnt = nat.empty((1,), np.int32)
    nat.call("rk_stride_compact", lm.device_sensor(intr), nat.ptr(rng), 1, int(stride),
             float(np.float32(clip_min)), float(np.float32(clip_max)), nat.ptr(idx), nat.ptr(cnt),
             nat.stream_ptr())
    n = int(cnt.item())
    return idx[:n], cnt


def _points_from_indices(img: RangeImage, idx, cnt):
    intr = _require_intrinsics(img)
    rng = img.device_data()
    n = idx.shape[0]
    out = nat.empty((n, 3), np.float64)
    if n:
        nat.call("rk_unproject_pixels", lm.device_sensor(intr), nat.ptr(rng), nat.ptr(idx),
                 nat.ptr(cnt), n, nat.ptr(out), nat.stream_ptr())
    return out


def to_point_cloud(img: RangeImage, clip_min: float = 0.0, clip_max: float = np.inf):
    """One float64 point per valid, clipped pixel, row-major (range_image.py:136-143)."""
    idx, cnt = stride_indices(img, 1, clip_min, clip_max)
    return _ret(img, _points_from_indices(img, idx, cnt))


def points_at_stride(img: RangeImage, stride: int, clip_min: float = 0.0,
                     clip_max: float = np.inf):
    """Cloud of the stride-decimated grid (range_image.py:146-157)."""
    if stride < 1:
        raise ValueError("stride must be >= 1")
    idx, cnt = stride_indices(img, stride, clip_min, clip_max)
    return _ret(img, _points_from_indices(img, idx, cnt))


@nvtx("compute_normal_map")
def compute_normal_map(img: RangeImage, method: str = "cross", radius: int = 2,
                       discontinuity_abs: float = DISCONTINUITY_ABS,
                       discontinuity_rel: float = DISCONTINUITY_REL) -> NormalImage:
    """Sensor-facing unit normals (range_image.py:197-212)."""
    if method == "cross":
        return normals_cross(img)
    if method == "pca":
        return normals_pca(img, radius, discontinuity_abs, discontinuity_rel)
    raise ValueError(f"unknown normal method {method!r}")


def normals_pca(img: RangeImage, radius: int = 2, discontinuity_abs: float = DISCONTINUITY_ABS,
                discontinuity_rel: float = DISCONTINUITY_REL) -> NormalImage:
    """Windowed-PCA normals (range_image.py:243-283): smallest covariance
    eigenvector over the valid neighbours of a (2*radius+1)^2 window that are
    not across a depth discontinuity; invalid with fewer than 3 of them."""
    intr = _require_intrinsics(img)
    rng = img.device_data()
    H, W = intr.height, intr.width
    vec = nat.empty((H, W, 3), np.float32)
    val = nat.empty((H, W), np.uint8)
    surf = nat.empty((H, W, 4), np.float32)
    nat.call("rk_normals_pca", lm.device_sensor(intr), nat.ptr(rng), 1, int(radius),
             float(discontinuity_abs), float(discontinuity_rel), nat.ptr(vec), nat.ptr(val),
             nat.ptr(surf), nat.stream_ptr())
    if img.on_device:
        return NormalImage(vec, val.bool(), surf)
    return NormalImage(nat.to_host(vec), nat.to_host(val).astype(bool), surf)


def normals_cross(img: RangeImage) -> NormalImage:
    """K1 (range_image.py:221-240), bit-exact float64 restatement."""
    intr = _require_intrinsics(img)
    rng = img.device_data()
    H, W = intr.height, intr.width
    vec = nat.empty((H, W, 3), np.float32)
    val = nat.empty((H, W), np.uint8)
    surf = nat.empty((H, W, 4), np.float32)
    nat.call("rk_normals_cross", lm.device_sensor(intr), nat.ptr(rng), 1, nat.ptr(vec),
             nat.ptr(val), nat.ptr(surf), nat.stream_ptr())
    if img.on_device:
        return NormalImage(vec, val.bool(), surf)
    return NormalImage(nat.to_host(vec), nat.to_host(val).astype(bool), surf)


@dataclass
class SurfelPyramid:
    """Per image: the full surfel map followed by the decimated map of every
    coarse stride (rk_normals_cross_pyramid), as 16-byte records {nx, ny,
    nz, range-if-valid} (32-byte builds append {target x, y, z, 0});
    ``offsets`` maps stride -> pixel offset inside an image's ``pitch``-pixel
    block (stride 1 -> 0)."""

    data: object
    pitch: int
    offsets: dict


@nvtx("normals_cross_batch")
def normals_cross_batch(intr: LidarIntrinsics, ranges, strides=None):
    """K1 over a (B, H, W) device batch -> (B, H, W, 4) surfel maps (batch
    API), or with ``strides`` a SurfelPyramid whose coarse levels the
    registration gathers from compact maps."""
    H, W = intr.height, intr.width
    t = nat.torch()
    if not (nat.is_tensor(ranges) and ranges.is_cuda and ranges.dtype == t.float32 and ranges.ndim == 3
            and tuple(ranges.shape[1:]) == (H, W) and ranges.is_contiguous()):
        raise ValueError(f"ranges must be a contiguous (B, {H}, {W}) float32 CUDA tensor")
    B = ranges.shape[0]
    if strides is None:
        surf = nat.empty((B, H, W, 4), np.float32)
        nat.call("rk_normals_cross", lm.device_sensor(intr), nat.ptr(ranges), B, None, None,
                 nat.ptr(surf), nat.stream_ptr())
        return surf
    coarse = sorted({int(s) for s in strides if int(s) > 1})
    offsets, off = {1: 0}, H * W
    for s in coarse:
        offsets[s] = off
        off += -(-H // s) * -(-W // s)
    pitch = off
    data = nat.empty((B, pitch, nat.load().rk_surfel_record_floats()), np.float32)
    st = np.asarray(coarse, dtype=np.int32)
    nat.call("rk_normals_cross_pyramid", lm.device_sensor(intr), nat.ptr(ranges), B,
             st.ctypes.data if st.size else None, int(st.size), nat.ptr(data), int(pitch),
             nat.stream_ptr())
    return SurfelPyramid(data, pitch, offsets)


@dataclass
class ProjectionStats:
    """Bookkeeping from from_point_cloud (range_image.py:119-126)."""

    kept: int = 0
    collisions: int = 0
    out_of_fov: int = 0
    degenerate: int = 0


@nvtx("from_point_cloud")
def from_point_cloud(points, intr: LidarIntrinsics, max_iters: int = 3, tol: float = 1e-4):
    """Project a cloud into a fresh image, nearest range wins pixel collisions
    (range_image.py:170-194): the float64 projection (rk_project_f64) then a
    64-bit atomicMin z-buffer (rk_zbuffer_image).  Returns (RangeImage,
    ProjectionStats); the image stays on the device for device input."""
    on_dev = _is_dev(points)
    pts = nat.to_dev(points, np.float64).reshape(-1, 3)
    n = int(pts.shape[0])
    H, W = intr.height, intr.width
    sensor = lm.device_sensor(intr)
    st = nat.stream_ptr()
    u = nat.empty((max(n, 1),), np.float64)
    v = nat.empty((max(n, 1),), np.int32)
    r = nat.empty((max(n, 1),), np.float64)
    status = nat.empty((max(n, 1),), np.int8)
    if n:
        work = nat.empty((3 * n + 4,), np.float64)
        nat.call("rk_project_f64", sensor, nat.ptr(pts), n, int(max_iters), float(tol), 1,
                 nat.ptr(u), nat.ptr(v), nat.ptr(r), nat.ptr(status), nat.ptr(work), st)
    out = nat.empty((H, W), np.float32)
    stats = nat.zeros((4,), np.int64)
    zb = nat.empty((H * W,), np.int64)
    nat.call("rk_zbuffer_image", sensor, nat.ptr(u), nat.ptr(v), nat.ptr(r), nat.ptr(status), n,
             nat.ptr(out), nat.ptr(stats), nat.ptr(zb), st)
    k = [int(x) for x in nat.to_host(stats)]
    ps = ProjectionStats(kept=k[0], collisions=k[1], out_of_fov=k[2], degenerate=k[3])
    return RangeImage(out if on_dev else nat.to_host(out), intr), ps
