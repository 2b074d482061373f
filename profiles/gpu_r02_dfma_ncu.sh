#!/bin/bash
mkdir -p gpurun_out
KCG_SANITIZE_SMALL=1 timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tests/sanitize_gram.py > gpurun_out/r02_sanitize_gram_racecheck.log 2>&1; echo racecheck=$?; grep -E "SUMMARY" gpurun_out/r02_sanitize_gram_racecheck.log | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_gram_dfma --launch-skip 2 --launch-count 1 -o gpurun_out/r02_gram_dfma18 -f python profiles/time_gram.py 8000000 18 > gpurun_out/ncu_dfma.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_gram_dfma --launch-skip 2 --launch-count 1 -o gpurun_out/r02_gram_dfma9 -f python profiles/time_gram.py 8000000 9 > gpurun_out/ncu_dfma9.log 2>&1; echo ncu9=$?
