#!/bin/bash
# f1 device CFL: tests + bench (device loop vs host loop), and 2-D variant sweep
TAG=${1:-cfl}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_cfl_gpu.py tests/test_p2p_gpu.py -q -x > $OUT/pytest_cfl.log 2>&1; echo "rc=$?" >> $OUT/pytest_cfl.log
for w in cfl1024 cfl6400; do
  for l in device host; do
    timeout 300 python bench.py --workload $w --cfl-loop $l --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}_${l}.json 2>>$OUT/err.log
  done
done
for v in 37 44 46 47; do
  RPL_VARIANT=$v timeout 120 python bench.py --steps 50 --no-cpu-baseline --e2e-steps 0 > $OUT/b_v${v}.json 2>>$OUT/err.log
  RPL_VARIANT=$v timeout 300 python bench.py --workload p6400 --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_p6400_v${v}.json 2>>$OUT/err.log
done
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{os.path.basename(f):26s} {d['value']:7.2f} Gcell/s {d['ms_per_step']*1e3:9.1f} us/step {d['roofline']['launch_ms']*1e3:9.1f} us/launch frac {d['roofline']['frac']:.3f}")
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/summary.txt; tail -3 $OUT/pytest_cfl.log; tail -3 $OUT/pytest_all.log
