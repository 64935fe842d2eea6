import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs librkb200.so kernels")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class Golden:
    """Lazy access to tests/golden/<file>.npz written by make_golden.py."""

    def __init__(self, name):
        self._z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)

    def __getitem__(self, k):
        return self._z[k]

    def __contains__(self, k):
        return k in self._z.files


@pytest.fixture(scope="session")
def golden_proj():
    return Golden("sensor_projection")


@pytest.fixture(scope="session")
def golden_icp():
    return Golden("images_icp")


@pytest.fixture(scope="session")
def golden_tsdf():
    return Golden("tsdf")


@pytest.fixture(scope="session")
def golden_mesh():
    return Golden("mesh")


@pytest.fixture(scope="session")
def golden_next():
    return Golden("next")


@pytest.fixture(scope="session")
def sensors():
    from paper_2112_02779_b200 import scenes
    return {"small": scenes.small_calib(), "synth": scenes.synth_intr(), "ouster": scenes.ouster64()}


@pytest.fixture(scope="session")
def osensors(sensors):
    from oracle.sensor import Sensor
    return {k: Sensor.from_intrinsics(v) for k, v in sensors.items()}


@pytest.fixture
def fast_math():
    """Run a test in MATH_FAST (the opt-in tolerance-contract mode; the
    default MATH_NP has its own bit-exact tests, test_gpu_numpy_exact.py)."""
    from paper_2112_02779_b200 import lidar_model as lm
    with lm.math_mode(lm.MATH_FAST):
        yield
