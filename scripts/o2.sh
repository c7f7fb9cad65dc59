#!/bin/bash
TAG=${1:-o2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_order2_gpu.py tests/test_cfl_gpu.py -q > $OUT/pytest_o2.log 2>&1; echo "rc=$?" >> $OUT/pytest_o2.log
tail -5 $OUT/pytest_o2.log
for v in 0 71 72 73; do
  RPL_VARIANT=$v timeout 120 python bench.py --workload o2_1024 --steps 30 --no-cpu-baseline --e2e-steps 0 > $OUT/b_o2_v${v}.json 2>>$OUT/err.log
done
timeout 120 python bench.py --workload o2_1024 --kernel split --steps 20 --no-cpu-baseline --e2e-steps 0 > $OUT/b_o2_split.json 2>>$OUT/err.log
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{os.path.basename(f):26s} {d['value']:7.2f} Gcell/s {d['ms_per_step']*1e3:9.1f} us/step {d['roofline']['launch_ms']*1e3:9.1f} us/launch frac {d['roofline']['frac']:.3f}")
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/summary.txt; tail -5 $OUT/err.log
