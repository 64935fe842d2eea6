#!/bin/bash
# The compute-sanitizer stand-in (the pool refuses compute-sanitizer): run the
# GPU suite, smoke() and a short bench with every extra against the
# RK_DEBUG_CHECKS=1 library (device bounds / invariant checks that trap).
#   python scripts/build_variants.py dbg:RK_DEBUG_CHECKS=1
#   gpurun -- 'bash scripts/gpu_debug_checks.sh'
set -u
mkdir -p gpurun_out
OUT=gpurun_out
export RK_LIB=$PWD/paper_2112_02779_b200/lib/librkb200_dbg.so
python - <<'PY'
import ctypes, os
lib = ctypes.CDLL(os.environ["RK_LIB"])
print("debug library:", os.environ["RK_LIB"])
PY
timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/dbg_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/dbg_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/dbg_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/dbg_smoke.log
timeout 900 python bench.py --steps 2 --warmup 3 --pairs 8192 --pool 512 --no-cpu > $OUT/dbg_bench.json 2> $OUT/dbg_bench.err; echo "bench rc=$?"
grep -h "RK_DCHECK\|illegal\|unspecified launch\|trap" $OUT/dbg_pytest.log $OUT/dbg_smoke.log $OUT/dbg_bench.err | head -20; echo "dcheck hits: $(cat $OUT/dbg_pytest.log $OUT/dbg_smoke.log $OUT/dbg_bench.err | grep -c RK_DCHECK)"
