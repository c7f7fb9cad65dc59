#!/bin/bash
# z-chunk length (planes per CTA march) sweep for the 3-D defaults
TAG=${1:-r2rows}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for w in ${WL:-s512 w384}; do
  for r in ${ROWS:-0 24 32 48 64 96 128}; do
    timeout 300 python bench.py --workload $w --extras none --rows $r --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}_$r.json 2>> $OUT/err
    python -c "import json; d=json.load(open('$OUT/b_${w}_$r.json')); r=d['roofline']; print('$w rows=$r', round(d['ms_per_step'],4), 'ms frac', round(r['frac'],3), d['clocks']['sm_mhz'])" >> $OUT/summary.txt 2>&1
  done
done
cat $OUT/summary.txt
