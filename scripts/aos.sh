#!/bin/bash
TAG=${1:-aos}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "aos or fused3d" > $OUT/pytest_aos.log 2>&1; echo "rc=$?" >> $OUT/pytest_aos.log
for dt in f32 f64; do for lay in soa aos; do
  timeout 300 python bench.py --workload l256 --dtype $dt --layout $lay --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_l256_${dt}_${lay}.json 2>>$OUT/err.log
  timeout 300 python bench.py --workload l256 --dtype $dt --layout $lay --kernel split --steps 5 --no-cpu-baseline --e2e-steps 0 > $OUT/b_l256_${dt}_${lay}_split.json 2>>$OUT/err.log
done; done
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
        print(f"{os.path.basename(f):28s} {d['value']:7.2f} Gcell/s {r['kernel']:9s} {r['launch_ms']*1e3:9.1f} us/launch frac {r['frac']:.3f}")
    except Exception as e: print(f, 'ERR', e)
PY
for dt in f32 f64; do for lay in soa aos; do
timeout 600 ncu --set full --clock-control none -k regex:k_step3d -s 3 -c 1 -o $OUT/ncu_l256_${dt}_${lay} python bench.py --workload l256 --dtype $dt --layout $lay --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done; done
cat $OUT/summary.txt
tail -2 $OUT/pytest_aos.log
