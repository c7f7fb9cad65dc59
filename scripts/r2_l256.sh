#!/bin/bash
# BASELINE configs[4]: 256^3, fp32 and fp64 x SoA and AoS, bench lines + ncu captures
OUT=gpurun_out/${1:-r2l256}; mkdir -p $OUT
for dt in f32 f64; do for lay in soa aos; do
  timeout 300 python bench.py --workload l256 --dtype $dt --layout $lay --extras none --steps 20 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${dt}_$lay.json 2>> $OUT/err
  python -c "import json; d=json.load(open('$OUT/b_${dt}_$lay.json')); r=d['roofline']; print('l256 $dt $lay', round(d['ms_per_step']*1e3,1), 'us', round(d['value'],2), 'Gcell/s frac', round(r['frac'],3), r['kernel'], d['clocks']['sm_mhz'])" >> $OUT/summary.txt
  timeout 600 ncu --set full --clock-control none -k regex:k_step3d -s 3 -c 1 -o $OUT/ncu_${dt}_$lay python bench.py --workload l256 --dtype $dt --layout $lay --extras none --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  timeout 300 python bench.py --workload l256 --dtype $dt --layout $lay --kernel split --extras none --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${dt}_${lay}_split.json 2>> $OUT/err
  python -c "import json; d=json.load(open('$OUT/b_${dt}_${lay}_split.json')); r=d['roofline']; print('l256 $dt $lay split', round(d['ms_per_step']*1e3,1), 'us', round(d['value'],2), 'Gcell/s', r['kernel'])" >> $OUT/summary.txt
done; done
cat $OUT/summary.txt
