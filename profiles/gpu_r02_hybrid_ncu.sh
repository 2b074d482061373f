#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_gram_hybrid --launch-skip 2 --launch-count 1 -o gpurun_out/r02_gram_hybrid -f python profiles/time_gram.py 8000000 40 > gpurun_out/ncu_hybrid.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_hybrid.log
