#!/bin/bash
TAG=${1:-dbg}
OUT=gpurun_out/$TAG
mkdir -p $OUT
VARS=60,61,62,63 timeout 900 python scripts/dbg_cm.py > $OUT/dbg_pp.txt 2>&1
for v in 34 60 61 62 63; do
  RPL_VARIANT=$v timeout 120 python bench.py --steps 50 --no-cpu-baseline --e2e-steps 0 > $OUT/b_v${v}.json 2>>$OUT/err.log
done
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(os.path.basename(f), round(d['value'],1), 'Gcell/s', round(d['ms_per_step']*1e3,2), 'us/step', round(d['roofline']['launch_ms']*1e3,2),'us', round(d['roofline']['frac'],3))
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/dbg_pp.txt $OUT/summary.txt
RPL_VARIANT=60 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step2d -s 3 -c 1 \
  -o $OUT/pp python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu.log 2>&1
