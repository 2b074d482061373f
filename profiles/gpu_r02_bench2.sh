#!/bin/bash
# Round 2 evidence: the default bench line, ncu of the default argmin build.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02_bench2.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/r02_bench2.log > gpurun_out/r02_bench2.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_multiam --launch-skip 2 --launch-count 1 -o gpurun_out/r02_argmin3 -f python profiles/time_argmin.py > gpurun_out/ncu_argmin3.log 2>&1; echo ncu=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_ref_arm.log 2>&1; echo ref_rc=$?; tail -1 gpurun_out/r02_ref_arm.log
