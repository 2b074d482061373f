#!/bin/bash
# Round-2 first call: the round-1 state on a fresh box (tests + default bench line).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt 2>&1
nproc > gpurun_out/r02_nproc.txt; lscpu | head -20 >> gpurun_out/r02_nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r02_gpu_tests.log
timeout 600 python bench.py > gpurun_out/r02_bench.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/r02_bench.log > gpurun_out/r02_bench.json
