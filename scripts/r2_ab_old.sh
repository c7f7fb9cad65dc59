#!/bin/bash
# A/B: current library vs scratch/libold.so (RPL_LIB) on the workloads in $WL
TAG=${1:-abold}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for w in ${WL:-p9600}; do
  for lib in new old; do
    if [ $lib = old ]; then export RPL_LIB=scratch/libold.so; else unset RPL_LIB; fi
    timeout 600 python bench.py --workload $w --steps ${STEPS:-50} --extras none --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}_$lib.json 2>> $OUT/err
    python -c "import json; d=json.load(open('$OUT/b_${w}_$lib.json')); print('$w $lib', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks'].get('sm_mhz'))" >> $OUT/summary.txt 2>&1
  done
done
unset RPL_LIB
for v in ${VARS:-}; do
  RPL_VARIANT=$v timeout 600 python bench.py --workload ${WL%% *} --steps ${STEPS:-50} --extras none --no-cpu-baseline --e2e-steps 0 > $OUT/b_v$v.json 2>> $OUT/err
  python -c "import json; d=json.load(open('$OUT/b_v$v.json')); print('${WL%% *} v$v', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3))" >> $OUT/summary.txt 2>&1
done
cat $OUT/summary.txt
