#!/bin/bash
# Full GPU test suite + smoke + bench lines of the 3-D/2-D configs (defaults)
TAG=${1:-r2check}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
for w in ${WL:-2d1024 s512 w384 l256}; do
  timeout 300 python bench.py --workload $w --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_$w.json 2>> $OUT/bench.err
done
for f in $OUT/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],2), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['roofline'].get('kernel'), d['clocks'].get('sm_mhz'))"; done > $OUT/summary.txt 2>&1
tail -3 $OUT/pytest_gpu.log; cat $OUT/smoke.log $OUT/summary.txt
