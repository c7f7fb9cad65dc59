#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over every step kernel (small grids)
# and the P2P flag kernel (2 processes sharing the GPU).
TAG=${1:-r2san}
OUT=gpurun_out/$TAG
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for c in 2d 3d64 3d32 o2 fd cfl split; do
    timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_driver.py $c > $OUT/${tool}_$c.log 2>&1
    echo "$tool $c rc=$?" >> $OUT/summary.txt
  done
done
# P2P transport: two ranks (processes) on one GPU, flag kernel + peer stores
timeout 900 $CS --tool memcheck --target-processes all --error-exitcode 9 python -m pytest tests/test_p2p_gpu.py -q -x -k "test_p2p_ranks_bitwise_equal_single_rank and n0" > $OUT/memcheck_p2p.log 2>&1
echo "memcheck p2p rc=$?" >> $OUT/summary.txt
timeout 900 $CS --tool synccheck --target-processes all --error-exitcode 9 python -m pytest tests/test_p2p_gpu.py -q -x -k "test_p2p_ranks_bitwise_equal_single_rank and n0" > $OUT/synccheck_p2p.log 2>&1
echo "synccheck p2p rc=$?" >> $OUT/summary.txt
cat $OUT/summary.txt
