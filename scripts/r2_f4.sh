#!/bin/bash
# f4: the paper's 2-D scaling problems on 1 B200, 1000 steps each, with clocks;
# the 8-way y-split tiling on one GPU (parts 1x8: the same decomposition as 8 ranks).
TAG=${1:-r2f4}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for w in p6400 p9600 pweak; do
  timeout 900 python bench.py --workload $w --extras none --steps 1000 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${w}_1000.json 2>> $OUT/bench.err
done
timeout 600 python -m pytest tests/test_parity_r2_gpu.py -q -k "p6400" > $OUT/pytest_p6400.log 2>&1; echo "rc=$?" >> $OUT/pytest_p6400.log
for f in $OUT/bench_*.json; do python -c "import json; d=json.load(open('$f')); r=d['roofline']; print('$f', d['steps'], round(d['value'],2), round(d['ms_per_step']*1e3,1), 'us', round(r['frac'],3), d['clocks'])"; done > $OUT/summary.txt 2>&1
cat $OUT/summary.txt; tail -2 $OUT/pytest_p6400.log
