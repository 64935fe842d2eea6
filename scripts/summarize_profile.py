#!/usr/bin/env python
"""Write the judged profile summaries under profiles/ from a GPU session's
gpurun_out/ artifacts.

    python scripts/summarize_profile.py TAG [--rep gpurun_out/prof_TAG.ncu-rep]
        [--launches gpurun_out/launches_TAG.csv]

Produces profiles/TAG_launches.md (per-kernel share of the ncu launch list,
cold-cache serialised timings) and profiles/TAG_ncu.md (one section per
captured kernel: duration, DRAM bytes, L2/L1 hit rates, issue activity, pipe
utilisation, stall mix), copying the raw launch CSV beside them.
"""
import argparse
import collections
import csv
import io
import shutil
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def launches(tag, path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    name, val = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        k = r[name].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        agg[k][0] += 1
        agg[k][1] += float(r[val].replace(",", ""))
    total = sum(t for _, t in agg.values())
    lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
             "Cold-cache, serialised per-launch times: compare SHARES, not absolutes, with bench.py.",
             "", "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {c} | {t / 1e3:.1f} | {t / c / 1e3:.2f} | {t / total:.1%} |")
    (PROF / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    shutil.copy(path, PROF / f"{tag}_launches.csv")


def full(tag, rep):
    rep = Path(rep)
    if rep.suffix == ".csv":   # the raw page exported on the GPU box (gpu_ncu.sh)
        rows = list(csv.reader(open(rep)))
    else:
        rows = ncu_csv(["-i", str(rep), "--page", "raw"])
    h, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(h)}
    out = [f"# {tag}: ncu --set full captures", "", f"Source: `{Path(rep).name}` (not committed; "
           "regenerate with scripts/gpu_profile.sh).", ""]
    stall_cols = [n for n in h if n.startswith("smsp__average_warps_issue_stalled_")
                  and n.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        try:
            inst = float(r[col["smsp__inst_executed.sum"]])
        except (ValueError, KeyError):
            continue
        if inst != inst:  # a replay that collected nothing (nan)
            continue
        out.append(f"## {r[col['Kernel Name']].split('(')[0]} (ID {r[col['ID']]})")
        out.append("")
        out.append("| metric | value |")
        out.append("|---|---|")
        for m, label in RAW:
            if m in col:
                out.append(f"| {label} | {r[col[m]]} {units[col[m]]} |")
        st = []
        for n in stall_cols:
            try:
                v = float(r[col[n]])
            except ValueError:
                continue
            if v >= 0.25:
                st.append((v, n.replace("smsp__average_warps_issue_stalled_", "")
                           .replace("_per_issue_active.ratio", "")))
        out.append("")
        out.append("Stall mix (warps stalled per issue): " +
                   ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)))
        out.append("")
    (PROF / f"{tag}_ncu.md").write_text("\n".join(out) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    a = ap.parse_args()
    PROF.mkdir(exist_ok=True)
    lp = Path(a.launches or ROOT / "gpurun_out" / f"launches_{a.tag}.csv")
    if lp.exists():
        launches(a.tag, lp)
    reps = [Path(a.rep)] if a.rep else (sorted((ROOT / "gpurun_out").glob(f"prof_*{a.tag}.ncu-rep"))
                                         or sorted((ROOT / "gpurun_out").glob(f"raw_*_{a.tag}.csv")))
    for rp in reps:
        name = rp.stem.replace("prof_", "").replace("raw_", "").replace(f"_{a.tag}", "")
        full(a.tag if name == a.tag else f"{a.tag}_{name}", rp)


if __name__ == "__main__":
    main()
