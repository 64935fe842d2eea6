#!/usr/bin/env python
"""Build experiment variants of librkb200.so in parallel:
    python scripts/build_variants.py name:DEF1=1,DEF2=0 name2:DEF=3 ...
-> paper_2112_02779_b200/lib/librkb200_<name>.so  (select with RK_LIB=...)."""
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def one(spec):
    import __graft_entry__ as g
    name, _, defs = spec.partition(":")
    out = ROOT / "paper_2112_02779_b200" / "lib" / f"librkb200_{name}.so"
    g.build(out=out, defines=tuple(d for d in defs.split(",") if d))
    return str(out)


if __name__ == "__main__":
    with ProcessPoolExecutor(len(sys.argv) - 1) as ex:
        for p in ex.map(one, sys.argv[1:]):
            print(p)
