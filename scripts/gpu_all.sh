#!/bin/bash
# tests + 2-D variants + 3-D benches (one gpurun call)
TAG=${1:-all}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for v in 0 10 32; do
  RPL_VARIANT=$v timeout 120 python bench.py --steps 50 --no-cpu-baseline --e2e-steps 0 > $OUT/b2d_v${v}.json 2>>$OUT/err.log
done
for w in l256 w384 s512; do
  timeout 300 python bench.py --workload $w --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}.json 2>>$OUT/err.log
done
RPL_VARIANT=20 timeout 300 python bench.py --workload w384 --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_w384_v20.json 2>>$OUT/err.log
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
        print(f"{os.path.basename(f):20s} {d['value']:8.2f} Gcell/s  {r['kernel']:9s} {r['launch_ms']*1e3:9.1f} us/launch  frac {r['frac']:.3f}")
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/summary.txt
tail -3 $OUT/pytest_gpu.log
