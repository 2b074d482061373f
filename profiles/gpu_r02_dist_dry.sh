#!/bin/bash
# Two-rank dry run of the bench's multi-rank path on one B200 (gloo: both
# ranks share cuda:0) -- the torchrun launch the driver uses for N > 1.
mkdir -p gpurun_out
KCG_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02_dist_dry.log 2>&1; echo dry_rc=$?
tail -1 gpurun_out/r02_dist_dry.log | cut -c1-400
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r02_dist_ref.log 2>&1; echo ref_rc=$?
tail -1 gpurun_out/r02_dist_ref.log | cut -c1-300
