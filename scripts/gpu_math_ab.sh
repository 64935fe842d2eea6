#!/bin/bash
# A/B of the projection arithmetic modes on a mid-size bench config
# (MATHS="fast np cr", PAIRS, POOL, FRAMES).  Outputs -> gpurun_out/math_<m>.json
set -u
mkdir -p gpurun_out
OUT=gpurun_out
SMALL="--steps 3 --warmup 3 --pairs ${PAIRS:-16384} --pool ${POOL:-1024} --frames ${FRAMES:-100} --no-cpu --no-e2e"
for m in ${MATHS:-fast np}; do
  timeout 300 python bench.py $SMALL --math $m > $OUT/math_$m.json 2> $OUT/math_$m.err
  echo -n "math $m rc=$? "
  python -c "import json; d=json.load(open('$OUT/math_$m.json')); print('reg/s', round(d['value']), 'K3 ms', round(d['phase_ms']['register'],2), 'frac', round(d['roofline']['frac'],4), 'tsdf fps', round(d['tsdf']['value']), 'tsdf ms', round(d['phase_ms']['tsdf_sequence'],3), 'gt', d['gt_recovered_frac'])" 2>&1 | tail -1
done
