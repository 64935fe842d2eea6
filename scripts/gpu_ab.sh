#!/bin/bash
# A/B of librkb200 variants x math modes (scripts/build_variants.py ->
# lib/librkb200_<v>.so; "base" = lib/librkb200.so), optionally after the GPU
# parity tests on the default build.
#   SPECS="base:np ahead0:np base:fast" PAIRS=16384 NOTEST=1 bash scripts/gpu_ab.sh
set -u
mkdir -p gpurun_out
OUT=gpurun_out
if [ -z "${NOTEST:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -q -rf -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 $OUT/pytest_gpu.log
fi
SMALL="--steps ${STEPS:-3} --warmup 3 --pairs ${PAIRS:-16384} --pool ${POOL:-1024} --frames ${FRAMES:-100} --no-cpu --no-e2e ${EXTRA:-}"
for rep in $(seq 1 ${REPS:-1}); do
for spec in ${SPECS:-base:np}; do
  v=${spec%%:*}; m=${spec##*:}
  if [ "$v" = "base" ]; then lib=$PWD/paper_2112_02779_b200/lib/librkb200.so; else lib=$PWD/paper_2112_02779_b200/lib/librkb200_$v.so; fi
  RK_LIB=$lib timeout 300 python bench.py $SMALL --math $m > $OUT/ab_${v}_$m.json 2> $OUT/ab_${v}_$m.err
  echo -n "$v/$m rc=$? "
  python -c "import json; d=json.load(open('$OUT/ab_${v}_$m.json')); print('reg/s', round(d['value']), 'K1 ms', round(d['phase_ms']['normals'],3), 'K3 ms', round(d['phase_ms']['register'],2), 'frac', round(d['roofline']['frac'],4), 'tsdf fps', round(d['tsdf']['value']), 'tsdf ms', round(d['phase_ms']['tsdf_sequence'],3), 'gt', d['gt_recovered_frac'])" 2>&1 | tail -1
done
done
