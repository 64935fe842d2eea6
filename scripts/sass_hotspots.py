#!/usr/bin/env python
"""Summarise an ncu SASS source page (``ncu -i X.ncu-rep --page source --csv
--print-source sass --kernel-name regex:K``): total executed warp
instructions, the hottest instructions by stall samples, and the long-
scoreboard stalls per load.

    python scripts/sass_hotspots.py /tmp/sass.csv [top]
"""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    col = {n: i for i, n in enumerate(hdr)}
    body = [r for r in rows[2:] if len(r) == len(hdr)]

    def num(r, name):
        try:
            return float(r[col[name]])
        except (ValueError, KeyError):
            return 0.0

    tot_inst = sum(num(r, "Instructions Executed") for r in body)
    tot_samp = sum(num(r, "Warp Stall Sampling (All Samples)") for r in body)
    print(f"{len(body)} SASS lines, {tot_inst:.4g} warp instructions, {tot_samp:.0f} samples")
    stalls = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
    agg = {n: sum(num(r, n) for r in body) for n in stalls}
    print("stall mix:", ", ".join(f"{k[6:]} {v / tot_samp:.1%}" for k, v in
                                  sorted(agg.items(), key=lambda x: -x[1]) if v / tot_samp > 0.01))
    ranked = sorted(body, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]
    for r in ranked:
        s = num(r, "Warp Stall Sampling (All Samples)")
        main_stall = max(stalls, key=lambda n: num(r, n))
        print(f"{r[col['Address']][-5:]} {s / tot_samp:6.2%} {num(r, 'Instructions Executed'):10.3g} "
              f"{main_stall[6:]:12s} {r[col['Source']].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
