#!/bin/bash
# One GPU session: parity tests, A/B of ICP occupancy variants, full bench,
# ncu launch list + full capture of the two hot kernels.  Outputs -> gpurun_out/
set -u
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu.log
SMALL="--steps 3 --warmup 2 --pairs 16384 --pool 1024 --frames 20 --no-cpu --no-e2e"
for v in "" _minb2 _minb4; do
  RK_LIB=$PWD/paper_2112_02779_b200/lib/librkb200$v.so timeout 300 python bench.py $SMALL > $OUT/ab$v.json 2> $OUT/ab$v.err
  echo "variant '$v' rc=$?"; python -c "import json,sys; d=json.load(open('$OUT/ab$v.json')); print(d['value'], d['phase_ms'], d['roofline']['frac'], d['tsdf']['value'])"
done
timeout 900 python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err; echo "bench full rc=$?"
tail -c 3000 $OUT/bench_full.json
PROF="--steps 1 --warmup 1 --pairs 4096 --pool 512 --frames 10 --no-cpu --no-e2e"
timeout 300 python bench.py $PROF > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py $PROF > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python bench.py $PROF > $OUT/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_register|k_integrate" -s 0 -c 3 -o $OUT/prof_r1 python bench.py $PROF > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -5 $OUT/ncu_full.log
