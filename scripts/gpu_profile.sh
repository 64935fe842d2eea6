#!/bin/bash
# One GPU session: parity tests, smoke, full bench (+ reference arm), ncu
# launch list + full capture of the two hot kernels.  Outputs -> gpurun_out/
set -u
mkdir -p gpurun_out
OUT=gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_full_$TAG.json 2> $OUT/bench_full_$TAG.err; echo "bench full rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_full_$TAG.json')); print(round(d['value']), d['tsdf']['value'], d['roofline']['frac'], d['tsdf']['roofline']['frac'], d['e2e']['value'] if d['e2e'] else None, d['cpu_baseline']['value'] if d['cpu_baseline'] else None)"
if [ -n "${REF:-}" ]; then
  timeout 600 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "bench ref rc=$?"; tail -c 400 $OUT/bench_ref_$TAG.json
fi
PROF="--steps 1 --warmup 1 --pairs 4096 --pool 512 --frames 10 --no-cpu --no-e2e"
timeout 300 python bench.py $PROF > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv python bench.py $PROF > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python bench.py $PROF > $OUT/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_register|k_integrate" -s 0 -c 3 -o $OUT/prof_$TAG python bench.py $PROF > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 $OUT/ncu_full.log
