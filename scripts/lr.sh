#!/bin/bash
TAG=${1:-lr}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "variants_bitwise" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
bash scripts/tune.sh $TAG 2d1024:0 2d1024:80 2d1024:81 2d1024:82 2d1024:83 2d1024:84 p6400:0 p6400:80 p6400:81 p6400:84 p6400:44
