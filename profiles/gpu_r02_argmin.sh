#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multi.py tests/test_gpu_parity.py -k "multi or argmin" -m gpu -x -q > gpurun_out/r02_argmin_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r02_argmin_tests.log
python profiles/time_argmin.py
KCG_ARGMIN_LEGACY=1 python profiles/time_argmin.py
KCG_MULTI_CTAS=2 python profiles/time_argmin.py
KCG_MULTI_CTAS=3 KCG_MULTI_RING_KB=64 python profiles/time_argmin.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_multiam --launch-skip 2 --launch-count 1 -o gpurun_out/r02_argmin -f python profiles/time_argmin.py > gpurun_out/ncu_argmin.log 2>&1; echo ncu=$?
