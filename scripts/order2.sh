#!/bin/bash
TAG=${1:-o2b}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_order2_gpu.py tests/test_cfl_gpu.py -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
bash scripts/tune.sh $TAG o2_s256:0:--steps=10 "o2_s256:0:--steps=5 --kernel split" o2_1024:0
