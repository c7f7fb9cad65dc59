#!/bin/bash
# Variant sweep: RPL_VARIANT per workload (WLV="wl:v1,v2 ...")
TAG=${1:-r2var}
OUT=gpurun_out/$TAG
mkdir -p $OUT
WLV=${WLV:-2d1024:0,2,3,4 p6400:0,2,3,4 s512:0,1,3,4 w384:0,1}
for spec in $WLV; do
  w=${spec%%:*}; vs=${spec#*:}
  for v in ${vs//,/ }; do
    RPL_VARIANT=$v timeout 300 python bench.py --workload $w --steps ${STEPS:-10} --extras none --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}_v$v.json 2>> $OUT/bench.err
    python -c "import json; d=json.load(open('$OUT/b_${w}_v$v.json')); print('$w v$v', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3), d['roofline'].get('kernel'), d['clocks'].get('sm_mhz'))" >> $OUT/summary.txt 2>&1
  done
done
cat $OUT/summary.txt
