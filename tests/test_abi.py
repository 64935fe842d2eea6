"""The C-ABI boundary (CPU-only checks, no kernel launches)."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "rkb200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*int\s+(rk_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2112_02779_b200 import _native
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    from paper_2112_02779_b200 import _native
    assert set(declared_symbols()) == set(_native.SIGNATURES)


def test_load_and_version():
    from paper_2112_02779_b200 import _native
    lib = _native.load()
    assert lib.rk_version() == 1
    assert _native.last_error() == ""
    # the ctypes mirrors of the ABI structs match the library's layout
    import ctypes
    assert lib.rk_struct_size(0) == ctypes.sizeof(_native.SensorDesc)
    assert lib.rk_struct_size(1) == ctypes.sizeof(_native.IcpConfig)


def test_sm100a_sass_present():
    import shutil
    import subprocess

    from paper_2112_02779_b200 import _native
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_means_loud_failure():
    """The package has no CPU path: compute entry points raise without a GPU."""
    import torch

    import paper_2112_02779_b200 as rk
    from paper_2112_02779_b200 import scenes
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    intr = scenes.small_calib()
    with pytest.raises(rk.DeviceError):
        rk.project_many(np.ones((4, 3), np.float32), intr, single=True)
    with pytest.raises(rk.DeviceError):
        rk.compute_normal_map(rk.RangeImage(np.ones((32, 256), np.float32), intr))


def test_status_codes_map_to_reference_exceptions():
    from paper_2112_02779_b200 import errors
    text = HEADER.read_text()
    codes = dict((name, int(v)) for name, v in re.findall(r"(RK_E\w+)\s*=\s*(-\d+)", text))
    assert codes["RK_EDEGENERATE_GEOM"] in errors.STATUS_TO_ERROR
    assert errors.STATUS_TO_ERROR[codes["RK_EDEGENERATE_GEOM"]] is errors.DegenerateGeometry
    assert errors.STATUS_TO_ERROR[codes["RK_EINVALID_POSE"]] is errors.InvalidPose
    assert errors.STATUS_TO_ERROR[codes["RK_EEMPTY"]] is errors.EmptyInput
    assert set(codes.values()) <= set(errors.STATUS_TO_ERROR)
