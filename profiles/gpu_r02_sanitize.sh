#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tests/sanitize_multi.py > gpurun_out/r02_sanitize_$tool.log 2>&1; echo $tool rc=$?; tail -2 gpurun_out/r02_sanitize_$tool.log
done
