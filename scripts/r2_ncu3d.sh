#!/bin/bash
# ncu full captures of the 3-D step kernels (one launch each)
TAG=${1:-r2ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for spec in "w384 ${V32:-91}" "s512 ${V64:-94}"; do
  set -- $spec
  RPL_VARIANT=$2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step3d -s 3 -c 1 \
    -o $OUT/ncu_$1_v$2 python bench.py --workload $1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_$1.log 2>&1
done
ls -la $OUT
