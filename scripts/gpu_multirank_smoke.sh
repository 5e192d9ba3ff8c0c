#!/bin/bash
# Multi-rank bench path on a single-GPU box: 2 ranks share cuda:0 over gloo (NCCL refuses duplicate devices).
mkdir -p gpurun_out
for c in c2 c5; do
  FFSAT_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --config $c --steps 20 --warmup 3 > gpurun_out/bench2_$c.json 2> gpurun_out/bench2_$c.err; echo bench2_$c=$?
  tail -3 gpurun_out/bench2_$c.err
done
