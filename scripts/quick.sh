#!/bin/bash
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python bench.py --steps 100 > $OUT/bench.json 2> $OUT/bench.err
for w in s512 w384; do
  timeout 300 python bench.py --workload $w --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}.json 2>>$OUT/bench.err
done
cat $OUT/bench.json
