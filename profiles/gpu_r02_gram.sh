#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gram" > gpurun_out/r02_gram_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r02_gram_tests.log
python profiles/time_gram.py 100000000 32,40,48
KCG_DMMA_GENERIC=1 python profiles/time_gram.py 100000000 32,40,48
python profiles/time_argmin.py
KCG_MULTIAM_CTAS=4 KCG_MULTIAM_RING_KB=48 python profiles/time_argmin.py
KCG_MULTIAM_CTAS=2 KCG_MULTIAM_RING_KB=96 python profiles/time_argmin.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_gram_dmma --launch-skip 2 --launch-count 1 -o gpurun_out/r02_gram_dmma -f python profiles/time_gram.py 8000000 40 > gpurun_out/ncu_gram.log 2>&1; echo ncu=$?
