#!/bin/bash
TAG=${1:-p2p}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_p2p_gpu.py -q -x > $OUT/p2p.log 2>&1; echo "rc=$?" >> $OUT/p2p.log
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/p2p.log $OUT/pytest_gpu.log
