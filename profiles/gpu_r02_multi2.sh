#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multi.py -m gpu -x -q > gpurun_out/r02_multi_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r02_multi_tests.log
python profiles/time_multi.py 551 --sep
for c in 3 1; do KCG_MULTI_CTAS=$c python profiles/time_multi.py; done
KCG_MULTI_CTAS=3 KCG_MULTI_RING_KB=64 python profiles/time_multi.py
KCG_MULTI_TILE_Q=2 python profiles/time_multi.py
KCG_MULTI_SHARE=0 python profiles/time_multi.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_multi --launch-skip 2 --launch-count 1 -o gpurun_out/r02_multi2 -f python profiles/time_multi.py 300 > gpurun_out/ncu_multi.log 2>&1; echo ncu=$?
