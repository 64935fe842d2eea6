#!/usr/bin/env python
"""Co-resident K3 clusters the launcher assumes per cluster size and math
mode (rk_icp_cluster_capacity: the occupancy query behind the latency tier)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_02779_b200 import _native as nat  # noqa: E402

torch.zeros(1, device="cuda")
lib = nat.load()
for m, name in ((3, "np"), (0, "fast")):
    print(name, {c: lib.rk_icp_cluster_capacity(m, c) for c in (2, 4, 8, 16)})
