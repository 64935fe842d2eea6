"""Range-image and intrinsics loading (io_formats.py:45-102)
against the reference's own outcomes on crafted payloads
(tests/golden/io.npz from tests/golden/make_golden_io.py): the decoded
ranges bit for bit, and for every malformed payload the same exception class
and the same reported byte offset.  Host-side parsing: runs without a GPU."""

from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden" / "io.npz"


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


def _names(gold, kind):
    return sorted({k.split("/")[1] for k in gold.files if k.startswith(kind + "/")})


def _outcome(fn):
    try:
        v = fn()
    except Exception as e:
        off = getattr(e, "offset", None)
        return type(e).__name__, -1 if off is None else int(off), None
    return "ok", -1, v


def _intr(hw):
    from paper_2112_02779_b200.lidar_model import LidarIntrinsics
    h, w = (int(x) for x in hw)
    return LidarIntrinsics(width=w, height=h, receiver_radius=0.0, azimuth_lut=np.zeros(h),
                           elevation_lut=np.linspace(-0.3, 0.2, h))


def test_rimg_cases_match_reference(gold, tmp_path):
    from paper_2112_02779_b200 import io_formats
    names = _names(gold, "rimg")
    assert len(names) >= 12
    for name in names:
        p = tmp_path / f"{name}.rimg"
        p.write_bytes(gold[f"rimg/{name}/blob"].tobytes())
        hw = gold[f"rimg/{name}/intr_hw"]
        intr = _intr(hw) if hw[0] >= 0 else None
        cls, off, v = _outcome(lambda: io_formats.read_range_image(p, intr))
        assert (cls, off) == (str(gold[f"rimg/{name}/cls"]), int(gold[f"rimg/{name}/offset"])), name
        if v is not None:
            ref = gold[f"rimg/{name}/data"]
            assert v.data.dtype == np.float32 and np.array_equal(v.data, ref), name


def test_rimg_write_read_round_trip(tmp_path):
    from paper_2112_02779_b200 import io_formats
    from paper_2112_02779_b200.range_image import RangeImage
    g = np.random.default_rng(0)
    data = g.uniform(0.0, 60.0, (16, 40)).astype(np.float32)
    data[g.random(data.shape) < 0.2] = 0.0
    p = tmp_path / "x.rimg"
    io_formats.write_range_image(p, RangeImage(data))
    blob = p.read_bytes()
    assert blob[:4] == b"RIMG" and len(blob) == 12 + 4 * data.size
    assert np.array_equal(io_formats.read_range_image(p).data, data)


def test_intrinsics_json_cases_match_reference(gold, tmp_path):
    from paper_2112_02779_b200 import io_formats
    for name in _names(gold, "json"):
        p = tmp_path / f"{name}.json"
        p.write_text(str(gold[f"json/{name}/text"]), encoding="utf-8")
        cls, off, v = _outcome(lambda: io_formats.read_intrinsics(p))
        assert (cls, off) == (str(gold[f"json/{name}/cls"]), int(gold[f"json/{name}/offset"])), name
        if v is not None:
            assert np.array_equal(np.asarray(v.ray_dirs), gold[f"json/{name}/ray_dirs"]), name
            assert np.array_equal(np.asarray(v.ray_origins), gold[f"json/{name}/ray_origins"]), name
            assert np.array_equal(np.asarray(v.fov_bounds, dtype=np.float64), gold[f"json/{name}/fov"]), name


def test_sample_pairs_matches_reference():
    """eval_metrics.sample_pairs (eval_metrics.py:57-70): the reference's
    outputs, recorded with
    PYTHONPATH=/root/reference/pkg/src python -c "from rangekit import eval_metrics as e;
    print(e.sample_pairs(20, 3, 5, seed=4), e.sample_pairs(6, 2, 9, seed=1))"."""
    from paper_2112_02779_b200 import pipeline
    from paper_2112_02779_b200.errors import EmptyInput
    assert pipeline.sample_pairs(20, 3, 5, seed=4) == [(8, 11), (9, 12), (13, 16), (14, 17), (15, 18)]
    assert pipeline.sample_pairs(6, 2, 9, seed=1) == [(0, 2), (1, 3), (2, 4), (3, 5)]
    with pytest.raises(EmptyInput):
        pipeline.sample_pairs(3, 3, 1)
    with pytest.raises(ValueError):
        pipeline.sample_pairs(10, 0, 1)
