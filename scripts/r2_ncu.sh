#!/bin/bash
# ncu full captures (one launch each) of the step kernels at the bench workloads,
# plus the launch list of the default bench command.
TAG=${1:-r2ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --extras none"
for w in ${WL:-s512 w384 2d1024 p6400}; do
  case $w in 2d*|p*) K=k_step2d;; *) K=k_step3d;; esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o $OUT/ncu_$w $B --workload $w > $OUT/ncu_$w.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_default.csv python bench.py --steps 3 --warmup 3 --extra-steps 3 \
  --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls -la $OUT
