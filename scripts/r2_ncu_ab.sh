#!/bin/bash
# ncu full capture of one step-kernel launch of workload $W with the current library
# and with scratch/libold.so (RPL_LIB), for an A/B comparison of kernel forms.
TAG=${1:-ncuab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --extras none"
for w in ${WL:-p6400}; do
  case $w in 2d*|p*) K=k_step2d;; *) K=k_step3d;; esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o $OUT/new_$w $B --workload $w > $OUT/new_$w.log 2>&1
  RPL_LIB=scratch/libold.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o $OUT/old_$w $B --workload $w > $OUT/old_$w.log 2>&1
done
ls -la $OUT
