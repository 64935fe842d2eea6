"""Goldens for MATH_NP's transcendentals: numpy's own float32 np.arctan2 /
np.arcsin (SVML on this AVX-512 host, the same numpy that produced every
other golden) over 4e6 seeded inputs each.  Stored: the SHA-1 of the full
outputs and the first 50,000 values (so a mismatch can be located).

    python tests/golden/make_golden_svml.py
"""

import hashlib
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT))
from svml_inputs import asin_inputs, atan2_inputs  # noqa: E402

KEEP = 50_000


def main():
    y, x = atan2_inputs()
    a = np.arctan2(y, x)
    q = asin_inputs()
    s = np.arcsin(q)
    assert a.dtype == np.float32 and s.dtype == np.float32
    np.savez_compressed(OUT / "svml.npz",
                        atan2_sha1=np.array(hashlib.sha1(a.tobytes()).hexdigest()),
                        asin_sha1=np.array(hashlib.sha1(s.tobytes()).hexdigest()),
                        atan2_head=a[:KEEP], asin_head=s[:KEEP],
                        numpy=np.array(np.__version__))
    print("wrote", OUT / "svml.npz")


if __name__ == "__main__":
    main()
