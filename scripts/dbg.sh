#!/bin/bash
TAG=${1:-dbg}
OUT=gpurun_out/$TAG
mkdir -p $OUT
./tools/dp_microbench > $OUT/dp.txt 2>&1
cat > /tmp/t3.py <<'PY'
import numpy as np, paper_2104_08571_b200 as R, workloads as W
n=(70,33,20); dx=[1/70]*3
U0=W.shock_bubble(n,dx=dx).astype(np.float32)
with R.Domain(n, dtype="f32", dx=dx, kernel="fused") as d:
    d.set_state(U0); d.advance(1e-4, 2); print(d.get_state().sum())
PY
PYTHONPATH=$PWD timeout 300 compute-sanitizer --tool memcheck python /tmp/t3.py > $OUT/sanitizer.txt 2>&1
CUDA_LAUNCH_BLOCKING=1 PYTHONPATH=$PWD timeout 300 python /tmp/t3.py > $OUT/t3.txt 2>&1
cuobjdump -sass paper_2104_08571_b200/libripple_fv.so | grep -c UTMALDG > $OUT/sass_utmaldg.txt
