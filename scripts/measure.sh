#!/bin/bash
# Round measurement: bench lines, reference arm, ncu launch list + full captures.
TAG=${1:-measure}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > $OUT/gpu.txt 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_reference.json 2>> $OUT/bench.err
timeout 300 python bench.py --kernel split --no-cpu-baseline --e2e-steps 0 > $OUT/bench_split.json 2>> $OUT/bench.err
for w in s512 w384 l256; do
  timeout 300 python bench.py --workload $w --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_$w.json 2>> $OUT/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $OUT/launches_2d1024.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step2d -s 3 -c 1 \
  -o $OUT/ncu_step2d python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_step2d.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step3d -s 3 -c 1 \
  -o $OUT/ncu_step3d_s512 python bench.py --workload s512 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_step3d.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step3d -s 3 -c 1 \
  -o $OUT/ncu_step3d_w384 python bench.py --workload w384 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_step3d_w.log 2>&1
ls -la $OUT
