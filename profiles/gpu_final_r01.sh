#!/bin/bash
# Round-1 bench line + ncu launch list + 2-rank functional dry run (gloo on one device)
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench_default.log > gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
  --log-file gpurun_out/launches_raw.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-fit > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
KCG_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e --no-cpu --fit-rows 100000000 > gpurun_out/dry2.log 2>&1; echo dry2_rc=$?; tail -1 gpurun_out/dry2.log | head -c 600; echo
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_arm.log 2>&1; echo ref_rc=$?; tail -1 gpurun_out/ref_arm.log | head -c 800
