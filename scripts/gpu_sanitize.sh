#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_probe.py
# (K4 CAS hash insert, K6 vertex publish, K3 cluster mode and batch mode).
# Logs -> gpurun_out/sanitize_<tool>_<mode>.log
set -u
mkdir -p gpurun_out
OUT=gpurun_out
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
$CS --version > $OUT/sanitize_version.log 2>&1; echo "compute-sanitizer rc=$?"
for tool in memcheck racecheck synccheck; do
  for mode in auto 0; do
    RK_ICP_CLUSTER=$mode timeout 900 $CS --tool $tool --error-exitcode 17 --print-limit 50 \
      python scripts/sanitize_probe.py > $OUT/sanitize_${tool}_${mode}.log 2>&1
    echo "sanitize $tool cluster=$mode rc=$?"; tail -3 $OUT/sanitize_${tool}_${mode}.log
  done
done
