#!/bin/bash
TAG=${1:-dbg}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python scripts/dbg_cm.py > $OUT/dbg_cm.txt 2>&1
for v in 0 50 51; do
  for w in s512 w384; do
    RPL_VARIANT=$v timeout 300 python bench.py --workload $w --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}_v$v.json 2>>$OUT/err.log
  done
done
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(os.path.basename(f), round(d['value'],1), 'Gcell/s', round(d['roofline']['launch_ms']*1e3,2),'us', round(d['roofline']['frac'],3))
    except Exception as e: print(f, 'ERR', e)
PY
