#!/bin/bash
# every bench workload once (short): nothing crashes with the current defaults
TAG=${1:-allwl}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for w in 2d1024 cfl1024 cfl6400 fd1k fd2k fd4k fd8k fd16k fd32k l256 o2_1024 o2_s256 p6400 p9600 pweak s512 w384; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/$w.json 2>> $OUT/err.log || echo "$w FAILED rc=$?" >> $OUT/fail.txt
done
timeout 300 python bench.py --workload cfl1024 --cfl-loop host --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/cfl1024_host.json 2>> $OUT/err.log || echo "cfl host FAILED" >> $OUT/fail.txt
timeout 300 python bench.py --kernel split --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/split.json 2>> $OUT/err.log || echo "split FAILED" >> $OUT/fail.txt
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{os.path.basename(f):20s} {d['value']:9.2f} {d['unit']:16s} {d['ms_per_step']*1e3:10.1f} us/step {d['roofline']['kernel']:16s} frac {d['roofline']['frac']:.3f} vs_baseline {d.get('vs_baseline')}")
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/summary.txt; cat $OUT/fail.txt 2>/dev/null
