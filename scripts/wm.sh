#!/bin/bash
TAG=${1:-wm}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "variants_bitwise" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
bash scripts/tune.sh $TAG 2d1024:0 2d1024:90 2d1024:91 2d1024:92 2d1024:93 2d1024:94 2d1024:95 p6400:0 p6400:90 p6400:94 p6400:95
