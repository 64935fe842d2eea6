#!/bin/bash
# A/B of librkb200 variants (scripts/build_variants.py -> lib/librkb200_<v>.so;
# "base" = lib/librkb200.so), after the GPU parity tests on the default build.
#   VARIANTS="base old m3" PAIRS=16384 bash scripts/gpu_ab.sh
set -u
mkdir -p gpurun_out
OUT=gpurun_out
if [ -z "${NOTEST:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -q -rf -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 $OUT/pytest_gpu.log
fi
SMALL="--steps 3 --warmup 3 --pairs ${PAIRS:-16384} --pool ${POOL:-1024} --frames ${FRAMES:-40} --no-cpu --no-e2e"
for v in ${VARIANTS:-base old}; do
  if [ "$v" = "base" ]; then lib=$PWD/paper_2112_02779_b200/lib/librkb200.so; else lib=$PWD/paper_2112_02779_b200/lib/librkb200_$v.so; fi
  RK_LIB=$lib timeout 300 python bench.py $SMALL > $OUT/ab_$v.json 2> $OUT/ab_$v.err
  echo -n "variant $v rc=$? "
  python -c "import json; d=json.load(open('$OUT/ab_$v.json')); print('reg/s', round(d['value']), 'K3 ms', round(d['phase_ms']['register'],2), 'frac', round(d['roofline']['frac'],4), 'tsdf fps', round(d['tsdf']['value']), 'tsdf ms', round(d['phase_ms']['tsdf_sequence'],3), 'gt', d['gt_recovered_frac'])" 2>&1 | tail -1
done
