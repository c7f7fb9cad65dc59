#!/bin/bash
TAG=${1:-promo}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for p in 0 1 2 3; do for w in s512 w384 l256; do
  RPL_L2PROMO=$p timeout 300 python bench.py --workload $w --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}_p$p.json 2>>$OUT/err.log
done; done
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
        print(f"{os.path.basename(f):28s} {d['value']:7.2f} Gcell/s {r['kernel']:9s} {r['launch_ms']*1e3:9.1f} us/launch frac {r['frac']:.3f}")
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/summary.txt
