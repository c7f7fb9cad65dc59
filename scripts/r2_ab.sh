#!/bin/bash
# Bench lines of the step configs first (quick perf read), then the full GPU suite + smoke.
TAG=${1:-r2ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
for w in ${WL:-s512 w384 2d1024 p6400}; do
  timeout 300 python bench.py --workload $w --steps ${STEPS:-10} --extras none --no-cpu-baseline --e2e-steps 0 > $OUT/bench_$w.json 2>> $OUT/bench.err
done
for f in $OUT/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],2), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['roofline'].get('kernel'), d['clocks'].get('sm_mhz'))"; done > $OUT/summary.txt 2>&1
cat $OUT/summary.txt
if [ -z "$NOTEST" ]; then
  timeout ${TTIME:-1500} python -m pytest tests -m gpu -x -q ${TESTS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
  tail -5 $OUT/pytest_gpu.log; cat $OUT/smoke.log
fi
