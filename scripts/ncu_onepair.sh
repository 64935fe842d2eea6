#!/bin/bash
# ncu --set full of one single-pair k_register launch (latency mode) with the
# source/SASS pages exported: LIB=<.so> CL=<RK_ICP_CLUSTER> TAG=<name>
set -u
mkdir -p gpurun_out
OUT=gpurun_out
RK_LIB=${LIB:-$PWD/paper_2112_02779_b200/lib/librkb200.so} RK_ICP_CLUSTER=${CL:-0} \
  ncu --set full --clock-control none --import-source on -k regex:k_register -s 2 -c 1 \
  -o $OUT/prof_one_$TAG -f python scripts/one_pair.py 4 > $OUT/ncu_one_$TAG.log 2>&1
ncu -i $OUT/prof_one_$TAG.ncu-rep --page raw --csv > $OUT/raw_one_$TAG.csv 2>/dev/null
ncu -i $OUT/prof_one_$TAG.ncu-rep --page source --csv --print-source sass > $OUT/sass_one_$TAG.csv 2>/dev/null
ncu -i $OUT/prof_one_$TAG.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src_one_$TAG.csv 2>/dev/null
rm -f $OUT/prof_one_$TAG.ncu-rep
