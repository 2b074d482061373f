#!/bin/bash
# One-pass multi-variant evaluate+predict: parity tests + knob A/B + ncu.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multi.py tests/test_host_io.py tests/test_capi.py -m gpu -x -q > gpurun_out/r02_multi_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r02_multi_tests.log
python profiles/time_multi.py 551 --sep
for c in 2 4; do KCG_MULTI_CTAS=$c python profiles/time_multi.py; done
KCG_MULTI_TILE_Q=2 python profiles/time_multi.py
KCG_MULTI_RING_KB=48 KCG_MULTI_CTAS=4 python profiles/time_multi.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_multi --launch-skip 2 --launch-count 1 -o gpurun_out/r02_multi -f python profiles/time_multi.py 300 > gpurun_out/ncu_multi.log 2>&1; echo ncu=$?
