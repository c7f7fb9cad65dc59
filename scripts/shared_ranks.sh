#!/bin/bash
# Functional run of the N>1 bench path with all ranks time-slicing ONE B200
# (RPL_SHARE_DEVICE=1, P2P transport): proves the multi-rank launch, halo stores
# and flag sync end to end.  Not scaling numbers (the ranks share one GPU).
TAG=${1:-shared}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for n in 2 4 8; do
  RPL_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29400 + n)) bench.py --gpus $n --steps 10 --warmup 3 \
    --transport p2p --no-cpu-baseline --e2e-steps 1 > $OUT/b_2d1024_n$n.json 2>> $OUT/err.log
done
RPL_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29410 bench.py --gpus 2 --workload w384 --steps 5 --warmup 3 \
  --transport p2p --no-cpu-baseline --e2e-steps 1 > $OUT/b_w384_n2.json 2>> $OUT/err.log
RPL_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29411 bench.py --gpus 2 --workload s512 --steps 3 --warmup 3 \
  --transport p2p --no-cpu-baseline --e2e-steps 1 > $OUT/b_s512_n2.json 2>> $OUT/err.log
for f in $OUT/*.json; do echo "== $f"; tail -c 700 $f; echo; done
tail -5 $OUT/err.log
