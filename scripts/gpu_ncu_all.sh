#!/bin/bash
# ncu --set full captures (one launch each) of every hot kernel on small bench
# configs, exported on the box as CSV pages (the reports embed the library's
# SASS and are too large to bring back).   TAG=r2u bash scripts/gpu_ncu_all.sh
set -u
mkdir -p gpurun_out
OUT=gpurun_out
TAG=${TAG:-prof}
cap() {  # name kernel-regex skip bench-args...
  local name=$1 k=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -f \
    -o $OUT/prof_${name}_$TAG python bench.py --no-cpu --no-e2e --no-extras "$@" > $OUT/ncu_full_${name}_$TAG.log 2>&1
  echo "ncu $name rc=$?"
  ncu -i $OUT/prof_${name}_$TAG.ncu-rep --page raw --csv > $OUT/raw_${name}_$TAG.csv 2>/dev/null
  ncu -i $OUT/prof_${name}_$TAG.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src_${name}_$TAG.csv 2>/dev/null
  rm -f $OUT/prof_${name}_$TAG.ncu-rep
}
SMALL="--steps 1 --warmup 1 --pairs 2048 --pool 512 --frames 12"
cap k_register k_register 0 $SMALL
cap k_normals k_normals_cross 0 $SMALL
cap k_integrate k_integrate 8 $SMALL
cap k_activate k_activate_image 8 $SMALL
cap k_integrate_c5 k_integrate 8 --steps 1 --warmup 1 --pairs 2048 --pool 512 --frames 12 --tsdf-config c5
cap k_mc_count k_mc_count 0 $SMALL
cap k_mc_vertices k_mc_vertices 0 $SMALL
ls -la $OUT/*_$TAG.csv | head -20
