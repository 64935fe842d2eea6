#!/bin/bash
# A/B of K3 variants (builds in paper_2112_02779_b200/lib/) x warps-per-pair, then parity tests.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu.log
SMALL="--steps 3 --warmup 2 --pairs 16384 --pool 1024 --frames 20 --no-cpu --no-e2e"
for v in ${VARIANTS:-"" _pf _m4 _m4pf}; do
  [ "$v" = "base" ] && v=""
  for w in ${WPPS:-8 4 2}; do
    RK_ICP_WPP=$w RK_LIB=$PWD/paper_2112_02779_b200/lib/librkb200$v.so timeout 300 python bench.py $SMALL > $OUT/ab$v.w$w.json 2> $OUT/ab$v.w$w.err
    echo -n "variant '$v' wpp=$w rc=$? "; python -c "import json,sys; d=json.load(open('$OUT/ab$v.w$w.json')); print(round(d['value']), round(d['phase_ms']['register'],2), round(d['roofline']['frac'],4), d['gt_recovered_frac'])"
  done
done
