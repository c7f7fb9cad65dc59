#!/bin/bash
TAG=${1:-r1z}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_cfl_gpu.py tests/test_order2_gpu.py -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for w in cfl1024 cfl6400; do
  timeout 300 python bench.py --workload $w --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/b_${w}_device.json 2>>$OUT/err.log
done
for k in 1 2 4 8 16; do
  timeout 600 python bench.py --workload fd${k}k --steps 20 --no-cpu-baseline --e2e-steps 3 > $OUT/b_fd${k}k.json 2>>$OUT/err.log
done
timeout 900 python bench.py --workload fd32k --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/b_fd32k.json 2>>$OUT/err.log
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{os.path.basename(f):26s} {d['value']:7.2f} {d['unit']:18s} {d['ms_per_step']*1e3:9.1f} us/step {d['roofline']['launch_ms']*1e3:9.1f} us/launch frac {d['roofline']['frac']:.3f} vs_paper {d.get('vs_baseline')}")
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/summary.txt; tail -3 $OUT/pytest.log; tail -5 $OUT/err.log
