#!/bin/bash
# Gram: parity tests (incl. the opt-in hybrid), timing of the default DMMA path
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gram" > gpurun_out/r02_hybrid_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r02_hybrid_tests.log
python profiles/time_gram.py 100000000 9,24,32,40,48
python profiles/time_gram.py 100000000 40
KCG_GRAM_HYBRID=1 python profiles/time_gram.py 100000000 40
