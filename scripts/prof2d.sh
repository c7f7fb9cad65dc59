#!/bin/bash
TAG=${1:-prof}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export RPL_VARIANT=${RPL_VARIANT:-4}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step2d -s 3 -c 1 \
  -o $OUT/step2d python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --rows 8 > $OUT/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 4 -c 1 \
  -o $OUT/sweep python bench.py --kernel split --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu2.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "3d or fused3d" > $OUT/pytest3d.log 2>&1; echo "rc=$?" >> $OUT/pytest3d.log
timeout 300 python bench.py --workload l256 --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/l256.json 2> $OUT/l256.err
timeout 300 python bench.py --workload s512 --steps 10 --no-cpu-baseline --e2e-steps 0 > $OUT/s512.json 2> $OUT/s512.err
timeout 300 python bench.py --workload s512 --kernel split --steps 5 --no-cpu-baseline --e2e-steps 0 > $OUT/s512_split.json 2>> $OUT/s512.err
ls -la $OUT
