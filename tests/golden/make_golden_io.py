"""Golden outcomes of the reference's range-image / intrinsics parsers
(io_formats.py:45-102, formats.md "RIMG"), produced by running the UNMODIFIED
reference on crafted payloads: valid files, and every validation branch with
the exception class and byte offset it reports.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_io.py

Runs only in the build container (needs /root/reference); writes
tests/golden/io.npz, which tests/test_io_golden.py checks the package against.
"""

from __future__ import annotations

import json
import os
import struct
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402

from rangekit import io_formats  # noqa: E402  (the reference)
from rangekit.lidar_model import LidarIntrinsics  # noqa: E402


def rimg(h, w, data=None):
    arr = np.zeros((h, w), "<f4") if data is None else np.asarray(data, "<f4").reshape(h, w)
    return b"RIMG" + struct.pack("<II", h, w) + arr.tobytes()


def rimg_cases():
    g = np.random.default_rng(5)
    ok = g.uniform(0.5, 40.0, (4, 6)).astype("<f4")
    ok[1, 2] = 0.0
    neg = ok.copy()
    neg[2, 3] = -1.0
    nan = ok.copy()
    nan[0, 1] = np.nan
    inf = ok.copy()
    inf[3, 5] = np.inf
    return {
        "valid": (rimg(4, 6, ok), None),
        "valid_intr": (rimg(4, 6, ok), (4, 6)),
        "bad_magic": (b"RIMX" + rimg(4, 6, ok)[4:], None),
        "short_magic": (b"RI", None),
        "header_incomplete": (b"RIMG\x04\x00\x00", None),
        "truncated_payload": (rimg(4, 6, ok)[:-5], None),
        "zero_height": (rimg(0, 6), None),
        "zero_width": (b"RIMG" + struct.pack("<II", 3, 0), None),
        "negative_value": (rimg(4, 6, neg), None),
        "nan_value": (rimg(4, 6, nan), None),
        "inf_value": (rimg(4, 6, inf), None),
        "intr_mismatch": (rimg(4, 6, ok), (4, 7)),
        "trailing_bytes": (rimg(4, 6, ok) + b"\x00\x01", None),
    }


def intr_for(hw):
    h, w = hw
    el = np.linspace(-0.3, 0.2, h)
    return LidarIntrinsics(width=w, height=h, receiver_radius=0.0, azimuth_lut=np.zeros(h),
                           elevation_lut=el)


def json_cases():
    h = 8
    el = np.deg2rad(np.linspace(-15.0, 15.0, h))
    az = np.deg2rad(np.resize([1.5, -1.5], h))
    calib = {"width": 64, "height": h, "receiver_radius_m": 0.02,
             "azimuth_offsets_rad": az.tolist(), "elevations_rad": el.tolist()}
    synth = {"width": 32, "height": 6, "mode": "synthetic", "fov_min_rad": -0.4, "fov_max_rad": 0.1}
    missing = dict(calib)
    del missing["receiver_radius_m"]
    bad_type = dict(calib, width="wide")
    return {
        "calibrated": json.dumps(calib),
        "synthetic": json.dumps(synth),
        "missing_key": json.dumps(missing),
        "bad_type": json.dumps(bad_type),
        "bad_json": '{"width": 64, "height": 8,, }',
        "not_sorted": json.dumps(dict(calib, elevations_rad=el[::-1].tolist())),
    }


def outcome(fn):
    try:
        v = fn()
    except Exception as e:  # the class name and offset are the contract
        off = getattr(e, "offset", None)
        return type(e).__name__, -1 if off is None else int(off), None
    return "ok", -1, v


def main():
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, (blob, hw) in rimg_cases().items():
            p = Path(d) / f"{name}.rimg"
            p.write_bytes(blob)
            intr = intr_for(hw) if hw else None
            cls, off, v = outcome(lambda: io_formats.read_range_image(p, intr))
            out[f"rimg/{name}/blob"] = np.frombuffer(blob, np.uint8)
            out[f"rimg/{name}/intr_hw"] = np.array(hw if hw else (-1, -1), np.int64)
            out[f"rimg/{name}/cls"] = np.array(cls)
            out[f"rimg/{name}/offset"] = np.array(off, np.int64)
            if v is not None:
                out[f"rimg/{name}/data"] = np.asarray(v.data, np.float32)
        for name, text in json_cases().items():
            p = Path(d) / f"{name}.json"
            p.write_text(text, encoding="utf-8")
            cls, off, v = outcome(lambda: io_formats.read_intrinsics(p))
            out[f"json/{name}/text"] = np.array(text)
            out[f"json/{name}/cls"] = np.array(cls)
            out[f"json/{name}/offset"] = np.array(off, np.int64)
            if v is not None:
                out[f"json/{name}/ray_dirs"] = np.asarray(v.ray_dirs, np.float64)
                out[f"json/{name}/ray_origins"] = np.asarray(v.ray_origins, np.float64)
                out[f"json/{name}/fov"] = np.asarray(v.fov_bounds, np.float64)
    np.savez_compressed(OUT / "io.npz", **out)
    for k in sorted(out):
        if k.endswith("/cls"):
            print(k, out[k], out[k.replace("/cls", "/offset")])


if __name__ == "__main__":
    main()
