#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + full capture of the step kernel.
# Usage (from this container): gpurun --timeout 1500 -- 'bash scripts/gpu_check.sh [tag]'
set -x
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --kernel split --no-cpu-baseline --e2e-steps 0 > $OUT/bench_split.json 2>> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step2d -s 5 -c 2 \
  -o $OUT/prof_step2d python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_full.log 2>&1
ls -la $OUT
