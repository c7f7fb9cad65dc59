#!/bin/bash
# Sweep fused 2-D kernel variants on one GPU (tuning; not a bench line).
TAG=${1:-tune}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for v in 2 3 4; do for r in 0 8 12 16 24 32; do
  RPL_VARIANT=$v timeout 120 python bench.py --steps 50 --no-cpu-baseline --e2e-steps 0 --rows $r > $OUT/b_v${v}_r${r}.json 2>>$OUT/err.log
done; done
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ.get('OUT','gpurun_out/tune')+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(os.path.basename(f), round(d['value'],1), 'Gcell/s', round(d['roofline']['launch_ms']*1e3,2),'us', round(d['roofline']['frac'],3))
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/summary.txt
