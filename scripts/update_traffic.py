#!/usr/bin/env python
"""profiles/traffic.json from one profile round's captures:

    python scripts/update_traffic.py TAG

DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and warp
instructions per algorithmic work unit for K3 (per source-point-iteration)
and K5 (per updated voxel), from profiles/TAG_k_*_ncu.md (one ncu --set full
launch each) and the work counts bench.py printed inside those same ncu runs
(gpurun_out/ncu_full_k_*_TAG.log).  bench.py reads the file for its
roofline.traffic and issue_roofline fields."""
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def metric(md, name):
    m = re.search(rf"^\| {re.escape(name)} \| ([0-9.e+]+) (\w+)", md, re.M)
    if not m:
        raise SystemExit(f"{name} missing")
    return float(m.group(1)) * UNIT.get(m.group(2), 1.0)


def main(tag):
    out = {}
    reg = (ROOT / "profiles" / f"{tag}_k_register_ncu.md").read_text()
    log = (ROOT / "gpurun_out" / f"ncu_full_k_register_{tag}.log").read_text()
    pt = float(re.search(r'"work": "([0-9.e+]+) source-point-iterations', log).group(1))
    dram = metric(reg, "DRAM read") + metric(reg, "DRAM write")
    ins = metric(reg, "warp instructions")
    out["k_register"] = round(dram / pt, 2)
    ins_reg = ins / pt
    note_reg = f"{dram / 1e9:.3f} GB and {ins:.4g} warp instructions over one launch of {pt:.4g} source-point-iterations"

    tsd = (ROOT / "profiles" / f"{tag}_k_integrate_ncu.md").read_text()
    log = (ROOT / "gpurun_out" / f"ncu_full_k_integrate_{tag}.log").read_text()
    upd = float(re.search(r'"voxels_updated_per_step": ([0-9.e+]+)', log).group(1))
    frames = int(re.search(r'"frames": ([0-9]+)', log).group(1))
    per_frame = upd / frames
    dram_t = metric(tsd, "DRAM read") + metric(tsd, "DRAM write")
    ins_t = metric(tsd, "warp instructions")
    out["k_integrate"] = round(dram_t / per_frame, 2)
    out["instructions"] = {"k_register": ins_reg, "k_integrate": ins_t / per_frame}
    out["_units"] = ("DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per algorithmic work unit; "
                     "'instructions': warp instructions (smsp__inst_executed.sum) per unit -- one ncu --set full "
                     f"launch each (profiles/{tag}_k_*_ncu.md)")
    out["_k_register"] = note_reg + " (bench --pairs 4096 --pool 512)"
    out["_k_integrate"] = (f"{dram_t / 1e6:.1f} MB and {ins_t:.4g} warp instructions over one frame of the "
                           f"{frames}-frame street sequence; per updated voxel using the sequence mean of "
                           f"{per_frame / 1e6:.2f} M updated voxels per frame (ncu flushes caches before the "
                           "launch, so the grid is read from DRAM here; in the bench it is mostly L2-resident)")
    (ROOT / "profiles" / "traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
