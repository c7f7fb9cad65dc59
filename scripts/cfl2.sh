#!/bin/bash
TAG=${1:-cfl2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_cfl_gpu.py tests/test_p2p_gpu.py -q > $OUT/pytest_cfl.log 2>&1; echo "rc=$?" >> $OUT/pytest_cfl.log
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
tail -3 $OUT/pytest_cfl.log; tail -3 $OUT/pytest_all.log
