#!/bin/bash
# One GPU session: parity tests, smoke, full bench (+ reference arm), ncu
# launch list of the bench command, and full ncu captures (one launch each)
# of the two hot kernels with their SASS source pages.  Outputs -> gpurun_out/
set -u
mkdir -p gpurun_out
OUT=gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -2 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_full_$TAG.json 2> $OUT/bench_full_$TAG.err; echo "bench full rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_full_$TAG.json')); print('reg/s', round(d['value']), 'tsdf fps', round(d['tsdf']['value']), 'frac', round(d['roofline']['frac'],4), round(d['tsdf']['roofline']['frac'],4), 'e2e', d['e2e']['value'] if d['e2e'] else None, 'cpu', d['cpu_baseline']['value'] if d['cpu_baseline'] else None)"
if [ -n "${REF:-}" ]; then
  timeout 600 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "bench ref rc=$?"; tail -c 300 $OUT/bench_ref_$TAG.json
fi
PROF="--steps 1 --warmup 1 --pairs 4096 --pool 512 --frames 20 --no-cpu --no-e2e"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv python bench.py $PROF > $OUT/ncu_launches_$TAG.log 2>&1; echo "ncu launches rc=$?"
for k in k_register k_integrate; do
  skip=0; [ $k = k_integrate ] && skip=10
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -f -o $OUT/prof_${k}_$TAG python bench.py $PROF > $OUT/ncu_full_${k}_$TAG.log 2>&1; echo "ncu $k rc=$?"
  ncu -i $OUT/prof_${k}_$TAG.ncu-rep --page source --csv --print-source sass > $OUT/sass_${k}_$TAG.csv 2>/dev/null
done
