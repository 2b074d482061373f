#!/bin/bash
# Gram: parity tests (default hybrid for even F in 34..40, the opt-in path), timing, ncu of the hybrid
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gram" > gpurun_out/r02_hybrid_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r02_hybrid_tests.log
python profiles/time_gram.py 100000000 34,38,40
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_gram_hybrid --launch-skip 2 --launch-count 1 -o gpurun_out/r02_gram_hybrid -f python profiles/time_gram.py 8000000 40 > gpurun_out/ncu_hybrid.log 2>&1; echo ncu=$?
