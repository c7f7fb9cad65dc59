#!/bin/bash
TAG=${1:-sp}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "variants_bitwise" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
bash scripts/tune.sh $TAG 2d1024:0 2d1024:50 2d1024:51 2d1024:52 2d1024:53 2d1024:54 2d1024:55 p6400:0 p6400:53 p6400:55 p6400:51
