#!/usr/bin/env python
"""Per-CUDA-source-line summary of an ncu source page exported with
``--page source --csv --print-source cuda,sass`` (gpu_ncu.sh src_*.csv):
instructions executed and stall samples per line.

    python scripts/src_hotspots.py gpurun_out/src_k_register_TAG.csv [top] [--by inst|samples]
"""
import csv
import sys


def main(path, top=30, by="inst"):
    rows = list(csv.reader(open(path)))
    cur, out = None, []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1]
            continue
        if len(r) > 8 and r[0].isdigit():
            try:
                samp, inst = float(r[4] or 0), float(r[7] or 0)
            except ValueError:
                continue
            out.append((samp, inst, cur.split("/")[-1], r[0], r[1][:100]))
    ts = sum(o[0] for o in out) or 1.0
    ti = sum(o[1] for o in out) or 1.0
    print(f"{ti:.4g} warp instructions, {ts:.0f} samples")
    key = (lambda o: -o[1]) if by == "inst" else (lambda o: -o[0])
    for o in sorted(out, key=key)[:top]:
        print(f"{o[1] / ti:6.2%} inst {o[0] / ts:6.2%} samp  {o[2]}:{o[3]} {o[4]}")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    by = "samples" if "--by" in sys.argv and sys.argv[sys.argv.index("--by") + 1] == "samples" else "inst"
    main(args[0], int(args[1]) if len(args) > 1 and args[1].isdigit() else 30, by)
