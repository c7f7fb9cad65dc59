#!/bin/bash
# f2 tiled flux-difference tile shapes (RPL_VARIANT 0/2/3), bitwise test + fd8k/fd16k benches
OUT=gpurun_out/${1:-r2vfd}; mkdir -p $OUT
for v in 0 2 3; do
  RPL_VARIANT=$v timeout 300 python -m pytest tests/test_parity_gpu.py tests/test_parity_r2_gpu.py -q -x -k "flux_difference_tiled or random_state_s15" >> $OUT/pytest.log 2>&1; echo "v=$v rc=$?" >> $OUT/pytest.log
  for w in fd8k fd16k; do for dt in f32 f64; do
    RPL_VARIANT=$v timeout 300 python bench.py --workload $w --dtype $dt --extras none --steps 20 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}_${dt}_v$v.json 2>> $OUT/err
    python -c "import json; d=json.load(open('$OUT/b_${w}_${dt}_v$v.json')); print('$w $dt v$v', round(d['ms_per_step']*1e3,1), 'us frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" >> $OUT/summary.txt
  done; done
done
cat $OUT/summary.txt; grep rc= $OUT/pytest.log
