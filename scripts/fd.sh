#!/bin/bash
TAG=${1:-fd}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_parity_gpu.py -q -k "flux_difference" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for k in 1 2 4 8 16; do
  timeout 600 python bench.py --workload fd${k}k --steps 20 --no-cpu-baseline --e2e-steps 3 > $OUT/b_fd${k}k.json 2>>$OUT/err.log
done
timeout 900 python bench.py --workload fd32k --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/b_fd32k.json 2>>$OUT/err.log
timeout 600 python bench.py --workload fd8k --kernel split --steps 20 --no-cpu-baseline --e2e-steps 0 > $OUT/b_fd8k_plain.json 2>>$OUT/err.log
ncu --set full --clock-control none --import-source on -k regex:k_fluxdiff_pt -s 3 -c 1 -o $OUT/fd8k python bench.py --workload fd8k --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu.log 2>&1
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{os.path.basename(f):22s} {d['value']:7.2f} {d['unit']:16s} {d['ms_per_step']*1e3:10.1f} us/step frac {d['roofline']['frac']:.3f} vs_paper_V100 {d.get('vs_baseline')}")
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/summary.txt; tail -3 $OUT/pytest.log; tail -3 $OUT/err.log
