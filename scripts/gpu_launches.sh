#!/bin/bash
# ncu launch list (gpu__time_duration) of a small bench run -> gpurun_out/launches_$TAG.csv
set -u
mkdir -p gpurun_out
TAG=${TAG:-ll}
CFG="--steps 1 --warmup 1 --pairs ${PAIRS:-2048} --pool 512 --frames ${FRAMES:-20} --no-cpu --no-e2e --no-extras"
timeout 300 python bench.py $CFG > gpurun_out/ll_plain_$TAG.json 2>&1 || { echo plain failed; tail -3 gpurun_out/ll_plain_$TAG.json; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py $CFG > gpurun_out/ll_ncu_$TAG.log 2>&1; echo "ncu rc=$?"
