#!/bin/bash
TAG=${1:-f4}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for w in p6400 p9600 pweak; do
  timeout 600 python bench.py --workload $w --steps 20 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}.json 2>>$OUT/err.log
  timeout 600 python bench.py --workload $w --steps 10 --kernel split --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}_split.json 2>>$OUT/err.log
done
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
        print(f"{os.path.basename(f):24s} {d['value']:7.2f} Gcell/s {d['ms_per_step']*1e3:9.1f} us/step {r['kernel']:12s} {r['launch_ms']*1e3:9.1f} us/launch frac {r['frac']:.3f}")
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/summary.txt
timeout 600 ncu --set full --clock-control none -k regex:k_step2d -s 3 -c 1 -o $OUT/ncu_p6400 python bench.py --workload p6400 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
