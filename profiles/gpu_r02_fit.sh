#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_tests_fit.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/r02_tests_fit.log
timeout 900 python bench.py > gpurun_out/r02_bench_fit.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/r02_bench_fit.log > gpurun_out/r02_bench_fit.json
