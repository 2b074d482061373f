#!/bin/bash
# narrow-design DFMA Gram + hybrid: parity tests, opt-in paths, compute-sanitizer, timing sweep
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gram" > gpurun_out/r02_dfma_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/r02_dfma_tests.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tests/sanitize_gram.py > gpurun_out/r02_sanitize_gram_$tool.log 2>&1; echo $tool=$?; tail -2 gpurun_out/r02_sanitize_gram_$tool.log
done
python profiles/time_gram.py 100000000 1,2,3,4,5,6,7,8,9,10,11,12,13,14,16,17,18,19,20,24,32,40
