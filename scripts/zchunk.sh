#!/bin/bash
# z-chunk (planes per CTA) sweep of the 3-D fused kernels (profiles/r1/rows_sweep.txt)
TAG=${1:-rows}
bash scripts/tune.sh $TAG "w384:0:--rows 24" "w384:0:--rows 32" "w384:0:--rows 40" "w384:0:--rows 48" \
  "s512:0:--rows 32" "s512:0:--rows 64" "s512:0:--rows 128" "s512:0" \
  "l256:0:--dtype f32 --rows 32" "l256:0:--dtype f32 --rows 48" "l256:0:--dtype f64 --rows 32" "l256:0:--dtype f64 --rows 64" "l256:0:--dtype f64"
