#!/bin/bash
# §7.3 flux-difference tile shapes: fp32 sizes x variants (0 default, 5 old 16-row x 4, 6 32-row), fp64 fd8k/fd16k
OUT=gpurun_out/${1:-r2fd}; mkdir -p $OUT
for w in fd1k fd2k fd4k fd8k fd16k fd32k; do for v in 0 5 6; do
  RPL_VARIANT=$v timeout 600 python bench.py --workload $w --steps 10 --extras none --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$w f32 v$v', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))" >> $OUT/summary.txt
done; done
for w in fd8k fd16k; do for v in 0 3 6; do
  RPL_VARIANT=$v timeout 600 python bench.py --workload $w --dtype f64 --steps 10 --extras none --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$w f64 v$v', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))" >> $OUT/summary.txt
done; done
cat $OUT/summary.txt
