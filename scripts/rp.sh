#!/bin/bash
# packed fp32 3-D kernel (k_step3d_rp): bitwise tests + benches vs the scalar kernel
TAG=${1:-rp}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "3d or minimum or fused3d" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python -m pytest tests/test_p2p_gpu.py -q -m gpu > $OUT/pytest_p2p.log 2>&1; echo "rc=$?" >> $OUT/pytest_p2p.log
tail -2 $OUT/pytest.log $OUT/pytest_p2p.log
bash scripts/tune.sh $TAG/t w384:0 w384:20 w384:71 "l256:0:--dtype f32" "l256:20:--dtype f32"
