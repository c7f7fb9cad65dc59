#!/bin/bash
# one full bench line (roofline + cpu_baseline + e2e) per SURVEY 8 row
TAG=${1:-rows}
OUT=gpurun_out/$TAG
mkdir -p $OUT
run() { name=$1; shift; timeout 900 python bench.py --extras none "$@" > $OUT/$name.json 2>>$OUT/err.log; }
run a_2d1024 --workload 2d1024
run a_s512 --workload s512 --steps 5 --e2e-steps 1
run a_w384 --workload w384 --steps 10 --e2e-steps 2
run a_l256_f32_soa --workload l256 --dtype f32 --layout soa --steps 20 --e2e-steps 2
run a_l256_f32_aos --workload l256 --dtype f32 --layout aos --steps 20 --e2e-steps 2
run a_l256_f64_soa --workload l256 --dtype f64 --layout soa --steps 20 --e2e-steps 2
run a_l256_f64_aos --workload l256 --dtype f64 --layout aos --steps 20 --e2e-steps 2
run f1_cfl1024_device --workload cfl1024 --steps 10 --e2e-steps 2
run f1_cfl1024_host --workload cfl1024 --cfl-loop host --steps 10 --e2e-steps 2
run f2_fd8k --workload fd8k --steps 20 --e2e-steps 2
run f3_o2_1024 --workload o2_1024 --steps 50 --e2e-steps 5
run f4_p6400 --workload p6400 --steps 10 --e2e-steps 1
run f4_p9600 --workload p9600 --steps 5 --e2e-steps 1
run f4_pweak --workload pweak --steps 10 --e2e-steps 1
OUT=$OUT python - <<'PY' > $OUT/summary.txt
import json,glob,os
for f in sorted(glob.glob(os.environ['OUT']+'/*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        cb=d.get('cpu_baseline') or {}
        e=d.get('e2e') or {}
        print(f"{os.path.basename(f):24s} {d['value']:8.2f} {d['unit']:16s} {d['ms_per_step']*1e3:10.1f} us/step {d['roofline']['kernel']:14s} frac {d['roofline']['frac']:.3f}  e2e {e.get('value',0):.3f}  cpu {cb.get('value',0):.4f} ({cb.get('cores')} core)  halo {d.get('halo',{}).get('exposed_ms_per_step')}")
    except Exception as ex: print(f, 'ERR', ex)
PY
cat $OUT/summary.txt; tail -3 $OUT/err.log
