#!/bin/bash
# compute-sanitizer over the Gram kernels incl. the integer-sliced tcgen05 Gram
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tests/sanitize_gram.py > gpurun_out/r02_sanitize_gram_$tool.log 2>&1; echo $tool=$?; grep -E "SUMMARY|gram ok" gpurun_out/r02_sanitize_gram_$tool.log | tail -2
done
KCG_SANITIZE_SMALL=1 timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tests/sanitize_gram.py > gpurun_out/r02_sanitize_gram_racecheck.log 2>&1; echo racecheck=$?; grep -E "SUMMARY|gram ok" gpurun_out/r02_sanitize_gram_racecheck.log | tail -2
