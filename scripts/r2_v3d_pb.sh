#!/bin/bash
TAG=${1:-r2pb}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "3d_kernel_variants" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 0 1 2 3; do
  RPL_VARIANT=$v timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "domain_error_is_reported_3d or minimum_sizes_fp32" >> $OUT/pytest_dom.log 2>&1; echo "v=$v rc=$?" >> $OUT/pytest_dom.log
done
for w in w384 s512; do
  for v in 0 1 2 3; do
    RPL_VARIANT=$v timeout 300 python bench.py --workload $w --extras none --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${w}_v$v.json 2>> $OUT/bench.err
    python -c "import json; d=json.load(open('$OUT/bench_${w}_v$v.json')); r=d['roofline']; print('$w v$v', round(d['ms_per_step'],4), 'ms frac', round(r['frac'],3), r['kernel'], d['clocks']['sm_mhz'])" >> $OUT/summary.txt 2>&1
  done
done
cat $OUT/summary.txt; tail -2 $OUT/pytest.log; grep rc= $OUT/pytest_dom.log
