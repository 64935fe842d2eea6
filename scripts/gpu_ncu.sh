#!/bin/bash
# ncu --set full capture of hot kernels on a small bench config (one launch
# each), plus the SASS source pages as CSV.
#   TAG=r2d MATH=np KERNELS="k_register k_integrate" LIB=... bash scripts/gpu_ncu.sh
set -u
mkdir -p gpurun_out
OUT=gpurun_out
TAG=${TAG:-prof}
LIB=${LIB:-$PWD/paper_2112_02779_b200/lib/librkb200.so}
CFG="--steps 1 --warmup 1 --pairs ${PAIRS:-2048} --pool 512 --frames 12 --no-cpu --no-e2e --math ${MATH:-np} ${EXTRA:-}"
RK_LIB=$LIB timeout 300 python bench.py $CFG > $OUT/ncu_plain_$TAG.json 2>&1 || { echo "plain run failed"; tail -5 $OUT/ncu_plain_$TAG.json; exit 1; }
for k in ${KERNELS:-k_register k_integrate}; do
  skip=0; [ $k = k_integrate ] && skip=8
  RK_LIB=$LIB timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -f -o $OUT/prof_${k}_$TAG python bench.py $CFG > $OUT/ncu_full_${k}_$TAG.log 2>&1; echo "ncu $k rc=$?"
  ncu -i $OUT/prof_${k}_$TAG.ncu-rep --page source --csv --print-source sass > $OUT/sass_${k}_$TAG.csv 2>/dev/null
  ncu -i $OUT/prof_${k}_$TAG.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src_${k}_$TAG.csv 2>/dev/null
  ncu -i $OUT/prof_${k}_$TAG.ncu-rep --page raw --csv > $OUT/raw_${k}_$TAG.csv 2>/dev/null
  # the reports embed the library's SASS (~45 MB): keep only the CSV pages
  [ -n "${KEEP:-}" ] || rm -f $OUT/prof_${k}_$TAG.ncu-rep
done
ls -la $OUT/*_$TAG.csv
