#!/bin/bash
# Round 2: 3-D kernel variants -- bitwise tests + bench sweep (w384 fp32, s512 fp64).
TAG=${1:-r2v3d}
VARS=${2:-"0 90 91 92 93 94"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "3d_kernel_variants or minimum_sizes_fp32 or fused3d" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in $VARS; do
  RPL_VARIANT=$v timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "domain_error_is_reported_3d" >> $OUT/pytest_dom.log 2>&1; echo "v=$v rc=$?" >> $OUT/pytest_dom.log
done
for w in w384 s512; do
  for v in $VARS; do
    RPL_VARIANT=$v timeout 300 python bench.py --workload $w --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${w}_v$v.json 2>> $OUT/bench.err
    python - $OUT/bench_${w}_v$v.json $v <<'PY' >> $OUT/summary.txt
import json,sys
try:
    d=json.load(open(sys.argv[1])); r=d['roofline']
    print(sys.argv[1].split('/')[-1], 'v', sys.argv[2], 'ms/step %.4f'%d['ms_per_step'], 'kernel_us %.1f'%(r.get('kernel_ms',0)*1000 if 'kernel_ms' in r else -1), 'frac %.3f'%r['frac'], d['clocks']['sm_mhz'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
  done
done
cat $OUT/summary.txt
