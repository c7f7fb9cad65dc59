#!/bin/bash
# A/B: current library vs $ALT (RPL_LIB) on the workloads in $WL
TAG=${1:-ablib}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for w in ${WL:-s512}; do
  for lib in cur alt cur alt; do
    if [ $lib = alt ]; then export RPL_LIB=$ALT; else unset RPL_LIB; fi
    timeout 600 python bench.py --workload $w --steps ${STEPS:-20} --extras none --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}_$lib.json 2>> $OUT/err
    python -c "import json; d=json.load(open('$OUT/b_${w}_$lib.json')); print('$w $lib', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks'].get('sm_mhz'))" >> $OUT/summary.txt 2>&1
  done
done
cat $OUT/summary.txt
