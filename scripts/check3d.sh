#!/bin/bash
TAG=${1:-check3d}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -n 3 $OUT/pytest_gpu.log
bash scripts/tune.sh $TAG/t w384:0 s512:0 "l256:0:--dtype f32" "l256:0:--dtype f32 --layout aos" "l256:0:--dtype f64" "l256:0:--dtype f64 --layout aos" 2d1024:0
