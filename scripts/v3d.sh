#!/bin/bash
TAG=${1:-v3d}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "3d_kernel_variants" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
bash scripts/tune.sh $TAG w384:0:--steps=10 w384:21:--steps=10 "l256:0:--dtype f32" "l256:21:--dtype f32" "l256:0:--dtype f64" "l256:21:--dtype f64" s512:0:--steps=5 s512:21:--steps=5
