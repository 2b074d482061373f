#!/bin/bash
# config-5 fit passes: timing + ncu --set full of the refinement-gradient kernel (kcg_rgrad_*)
mkdir -p gpurun_out
timeout 600 python profiles/time_fit5.py 1000 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rgrad --launch-skip 1 --launch-count 1 -o gpurun_out/r02_rgrad -f python profiles/time_fit5.py 400 > gpurun_out/ncu_rgrad.log 2>&1; echo ncu=$?
