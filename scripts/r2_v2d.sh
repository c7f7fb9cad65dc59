#!/bin/bash
TAG=${1:-r2v2d}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "2d_fused_bitwise or domain_error_is_reported" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for w in 2d1024 p6400 p9600; do
  for v in ${VARS:-0 1 2}; do
    RPL_VARIANT=$v timeout 300 python bench.py --workload $w --extras none --steps 20 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${w}_v$v.json 2>> $OUT/bench.err
    python -c "import json; d=json.load(open('$OUT/bench_${w}_v$v.json')); r=d['roofline']; print('$w v$v', round(d['ms_per_step']*1000,1), 'us frac', round(r['frac'],3), r['kernel'], d['clocks']['sm_mhz'])" >> $OUT/summary.txt 2>&1
  done
done
cat $OUT/summary.txt; tail -2 $OUT/pytest.log
