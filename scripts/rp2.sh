#!/bin/bash
TAG=${1:-rp2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
cap() { name=$1; regex=$2; shift 2; timeout 900 ncu --set full --clock-control none --import-source on -k regex:$regex -s 2 -c 1 -o $OUT/$name python bench.py --no-cpu-baseline --e2e-steps 0 --warmup 3 "$@" > $OUT/$name.log 2>&1;
  python tools/ncu_summary.py $OUT $name=$OUT/$name.ncu-rep > /dev/null 2>&1;
  python tools/sass_mix.py $OUT/$name.ncu-rep > $OUT/sass_mix_$name.txt 2>&1; }
cap w384rp k_step3d_rp --workload w384 --steps 2
bash scripts/tune.sh $TAG/t w384:0 "w384:0:--rows 48" "w384:0:--rows 64" "w384:0:--rows 192" "w384:0:--rows 384" "l256:0:--dtype f32"
cat $OUT/ncu_w384rp.txt; head -30 $OUT/sass_mix_w384rp.txt
