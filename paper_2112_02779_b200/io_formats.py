"""On-disk formats of the hot path's boundary -- drop-in subset of
rangekit/io_formats.py: intrinsics JSON, RIMG range images (the "range-image
load" API of the north star), SDFG grid snapshots and binary PLY meshes
(normative layouts: reference pkg/formats.md).  Parsing is host work; the
parsed image is uploaded once by the first device call.
"""

from __future__ import annotations

import json
import struct

import numpy as np

from .errors import FormatError, InvalidIntrinsics, TruncatedPayload
from .lidar_model import MODE_CALIBRATED, MODE_SYNTHETIC, LidarIntrinsics, synthetic_intrinsics
from .range_image import RangeImage
from .sdf_volume import BLOCK_EDGE, VoxelBlockGrid

RIMG_MAGIC = b"RIMG"
GRID_MAGIC = b"SDFG"


def write_intrinsics(path, intr: LidarIntrinsics) -> None:
    doc = {"width": intr.width, "height": intr.height,
           "receiver_radius_m": intr.receiver_radius,
           "azimuth_offsets_rad": intr.azimuth_lut.tolist(),
           "elevations_rad": intr.elevation_lut.tolist(), "mode": intr.mode}
    with open(path, "w", encoding="utf-8") as f:
        json.dump(doc, f, indent=1)
        f.write("\n")


def read_intrinsics(path) -> LidarIntrinsics:
    """io_formats.py:45-68."""
    with open(path, "r", encoding="utf-8") as f:
        try:
            doc = json.load(f)
        except json.JSONDecodeError as e:
            raise FormatError(f"intrinsics JSON: {e.msg}", offset=e.pos) from e
    try:
        mode = doc.get("mode", MODE_CALIBRATED)
        width, height = int(doc["width"]), int(doc["height"])
        if mode == MODE_SYNTHETIC and "elevations_rad" not in doc:
            return synthetic_intrinsics(height, width, float(doc["fov_min_rad"]),
                                        float(doc["fov_max_rad"]))
        return LidarIntrinsics(width=width, height=height,
                               receiver_radius=float(doc["receiver_radius_m"]),
                               azimuth_lut=np.asarray(doc["azimuth_offsets_rad"], dtype=float),
                               elevation_lut=np.asarray(doc["elevations_rad"], dtype=float),
                               mode=mode)
    except KeyError as e:
        raise FormatError(f"intrinsics JSON missing key {e.args[0]!r}") from e
    except (TypeError, ValueError) as e:
        raise FormatError(f"intrinsics JSON: {e}") from e


def write_range_image(path, img: RangeImage) -> None:
    with open(path, "wb") as f:
        f.write(RIMG_MAGIC)
        f.write(struct.pack("<II", img.height, img.width))
        f.write(np.asarray(img.data, dtype="<f4").tobytes())


def parse_range_image(blob: bytes, intr: LidarIntrinsics | None = None) -> np.ndarray:
    """Validate an RIMG payload (io_formats.py:80-102; formats.md RIMG)."""
    if blob[:4] != RIMG_MAGIC:
        raise FormatError(f"bad magic {blob[:4]!r}, expected {RIMG_MAGIC!r}", offset=0)
    if len(blob) < 12:
        raise TruncatedPayload("RIMG header incomplete", offset=len(blob))
    h, w = struct.unpack_from("<II", blob, 4)
    need = 12 + 4 * h * w
    if len(blob) < need:
        raise TruncatedPayload(f"RIMG declares {h}x{w} pixels ({need} bytes), file has {len(blob)}",
                               offset=len(blob))
    if h == 0 or w == 0:
        raise FormatError("RIMG dimensions must be positive", offset=4)
    data = np.frombuffer(blob, dtype="<f4", count=h * w, offset=12).reshape(h, w)
    bad = ~np.isfinite(data) | (data < 0)
    if bad.any():
        raise FormatError("non-finite or negative range value",
                          offset=12 + 4 * int(np.flatnonzero(bad)[0]))
    if intr is not None and (h, w) != (intr.height, intr.width):
        raise InvalidIntrinsics(f"image is {h}x{w}, intrinsics expect {intr.height}x{intr.width}")
    return data.astype(np.float32)


def read_range_image(path, intr: LidarIntrinsics | None = None) -> RangeImage:
    with open(path, "rb") as f:
        blob = f.read()
    return RangeImage(parse_range_image(blob, intr), intr)


_BLOCK_REC = np.dtype([("key", "<i4", (3,)), ("vox", "<f4", (BLOCK_EDGE ** 3, 2))])


def write_grid(path, grid: VoxelBlockGrid) -> None:
    """SDFG snapshot, blocks sorted by key (io_formats.py:267-277; formats.md
    "SDFG"): one bulk device read-back, one write."""
    keys, vox = grid.export_blocks()
    rec = np.empty(keys.shape[0], dtype=_BLOCK_REC)
    rec["key"] = keys
    rec["vox"] = vox
    with open(path, "wb") as f:
        f.write(GRID_MAGIC)
        f.write(struct.pack("<ddQ", grid.voxel_size, grid.truncation, keys.shape[0]))
        f.write(rec.tobytes())


def read_grid(path) -> VoxelBlockGrid:
    """io_formats.py:280-308: validation with byte offsets, then one bulk
    device upload."""
    with open(path, "rb") as f:
        blob = f.read()
    if blob[:4] != GRID_MAGIC:
        raise FormatError(f"bad magic {blob[:4]!r}, expected {GRID_MAGIC!r}", offset=0)
    if len(blob) < 28:
        raise TruncatedPayload("grid header incomplete", offset=len(blob))
    voxel, trunc, n = struct.unpack_from("<ddQ", blob, 4)
    if not (np.isfinite(voxel) and voxel > 0 and np.isfinite(trunc) and trunc > 0):
        raise FormatError("invalid voxel size or truncation", offset=4)
    per = _BLOCK_REC.itemsize
    if len(blob) < 28 + n * per:
        raise TruncatedPayload(f"grid declares {n} blocks", offset=len(blob))
    rec = np.frombuffer(blob, dtype=_BLOCK_REC, count=n, offset=28)
    bad = ~np.isfinite(rec["vox"][..., 0]).all(axis=1) | (rec["vox"][..., 1] < 0).any(axis=1)
    if np.any(bad):
        first = int(np.flatnonzero(bad)[0])
        raise FormatError("non-finite tsdf or negative weight in block", offset=28 + first * per + 12)
    grid = VoxelBlockGrid(voxel_size=voxel, truncation=trunc, capacity=max(1024, 2 * int(n)))
    grid.import_blocks(rec["key"], rec["vox"])
    return grid


def write_ply(path, mesh_or_points, normals=None) -> None:
    """Binary little-endian PLY (io_formats.py:169-199): float32 vertex records
    (+ normals), then uchar-count + 3 x int32 face records."""
    from .mesh_extract import TriangleMesh

    mesh = isinstance(mesh_or_points, TriangleMesh)
    verts = mesh_or_points.vertices if mesh else np.asarray(mesh_or_points, dtype=float).reshape(-1, 3)
    tris = mesh_or_points.triangles if mesh else None
    if mesh and normals is None:
        normals = mesh_or_points.normals
    fields = ["x", "y", "z"] + (["nx", "ny", "nz"] if normals is not None else [])
    vrec = np.empty(verts.shape[0], dtype=[(f, "<f4") for f in fields])
    cols = np.hstack([verts, normals]) if normals is not None else verts
    for i, f in enumerate(fields):
        vrec[f] = cols[:, i]
    lines = ["ply", "format binary_little_endian 1.0", f"element vertex {verts.shape[0]}"]
    lines += [f"property float {f}" for f in fields]
    if tris is not None:
        lines += [f"element face {tris.shape[0]}", "property list uchar int vertex_indices"]
    lines.append("end_header")
    payload = [("\n".join(lines) + "\n").encode("ascii"), vrec.tobytes()]
    if tris is not None and tris.shape[0]:
        frec = np.empty(tris.shape[0], dtype=[("n", "u1"), ("idx", "<i4", (3,))])
        frec["n"], frec["idx"] = 3, tris
        payload.append(frec.tobytes())
    with open(path, "wb") as f:
        f.write(b"".join(payload))
