#!/usr/bin/env python
"""List the loops (backward branches) of one kernel's SASS with their size and
the local-memory (LDL/STL) and global-load instructions inside -- a quick
check that the hot loop is spill-free before spending GPU time.

    cuobjdump -sass X.cubin | python scripts/sass_loops.py KERNEL_SUBSTRING
"""
import re
import sys

pat = sys.argv[1]
lines, on = [], False
for ln in sys.stdin:
    if "Function :" in ln:
        on = pat in ln
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if on and m:
        lines.append((int(m.group(1), 16), m.group(2).strip()))
addr = [a for a, _ in lines]
for a, ins in lines:
    b = re.search(r"BRA(?:\.\w+)* (?:`\()?\.?L?_?x?_?(0x[0-9a-f]+)", ins)
    if not b:
        continue
    tgt = int(b.group(1), 16)
    if tgt >= a:
        continue
    body = [i for aa, i in lines if tgt <= aa <= a]
    ldl = [i for i in body if i.split()[0].lstrip("@!P0123456789 ").startswith(("LDL", "STL"))
           or " LDL" in i or " STL" in i]
    ldg = sum(1 for i in body if "LDG" in i)
    mufu = sum(1 for i in body if "MUFU" in i)
    print(f"loop {tgt:#x}-{a:#x}: {len(body)} instr, {ldg} LDG, {mufu} MUFU, {len(ldl)} local:"
          f" {ldl[:6]}")
