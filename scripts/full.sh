#!/bin/bash
# round measurement: full GPU tests, smoke, default bench (+ reference arm), launch list,
# ncu of the headline step kernel
TAG=${1:-full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1
timeout 900 python bench.py > $OUT/bench_default.json 2>$OUT/bench_err.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2>>$OUT/bench_err.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_default.csv python bench.py --steps 2 --warmup 3 --extra-steps 2 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_step3d -s 3 -c 1 -o $OUT/step3d_s512 python bench.py --extras none --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_full.log 2>&1
tail -3 $OUT/pytest_gpu.log; cat $OUT/smoke.log | tail -1; cat $OUT/bench_default.json | tail -1 | cut -c1-400
