#!/bin/bash
TAG=${1:-tune}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "flux_difference" > $OUT/pytest_fd.log 2>&1; echo "rc=$?" >> $OUT/pytest_fd.log
for v in 34 37 38 39 30; do
  RPL_VARIANT=$v timeout 120 python bench.py --steps 50 --no-cpu-baseline --e2e-steps 0 > $OUT/b_v${v}.json 2>>$OUT/err.log
  RPL_VARIANT=$v timeout 300 python bench.py --workload p6400 --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_p6400_v${v}.json 2>>$OUT/err.log
done
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{os.path.basename(f):22s} {d['value']:7.2f} Gcell/s {d['ms_per_step']*1e3:9.1f} us/step {d['roofline']['launch_ms']*1e3:9.1f} us/launch frac {d['roofline']['frac']:.3f}")
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/summary.txt; tail -2 $OUT/pytest_fd.log
