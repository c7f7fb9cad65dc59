#!/bin/bash
TAG=${1:-r3d}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
bash scripts/tune.sh $TAG 2d1024:0 p6400:0 s512:0:--steps=5 w384:0:--steps=10 "l256:0:--layout aos --dtype f32" "l256:0:--layout soa --dtype f32" "l256:0:--layout soa --dtype f64" o2_1024:0
