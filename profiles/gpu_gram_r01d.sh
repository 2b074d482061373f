#!/bin/bash
# ncu --set full of the materialised DMMA Gram (config-3 shape, F = 40) and timing
mkdir -p gpurun_out
python profiles/time_gram.py 100000000 40,24,9
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_dmma --launch-skip 1 --launch-count 1 \
  -o gpurun_out/r01_gram_dmma -f python profiles/profile_kernels.py gram > gpurun_out/ncu_gram.log 2>&1; echo ncu_gram=$?
