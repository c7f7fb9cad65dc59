#!/bin/bash
# usage: tune.sh TAG "workload:variant[:extra args]" ...
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for spec in "$@"; do
  IFS=: read -r w v extra <<< "$spec"
  tag=$(echo "$extra" | tr -c 'a-z0-9' '_' | sed 's/_*$//')
  RPL_VARIANT=$v timeout 300 python bench.py --workload $w --steps 30 --no-cpu-baseline --e2e-steps 0 $extra > $OUT/b_${w}_v${v}${tag:+_$tag}.json 2>>$OUT/err.log
done
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/b_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{os.path.basename(f):28s} {d['value']:7.2f} {d['unit']:16s} {d['ms_per_step']*1e3:9.1f} us/step {d['roofline']['launch_ms']*1e3:9.1f} us/launch frac {d['roofline']['frac']:.3f}")
    except Exception as e: print(f, 'ERR', e)
PY
cat $OUT/summary.txt; tail -3 $OUT/err.log
