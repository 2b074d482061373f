#!/bin/bash
mkdir -p gpurun_out
python profiles/time_fit5.py 1000
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_rgrad --launch-skip 1 --launch-count 1 -o gpurun_out/r02_rgrad -f python profiles/time_fit5.py 400 > gpurun_out/ncu_rgrad.log 2>&1; echo ncu=$?
