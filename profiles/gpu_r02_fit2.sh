#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -m gpu -x -q -k "fit or dist or cli" > gpurun_out/r02_tests_fit2.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/r02_tests_fit2.log
timeout 900 python bench.py --no-e2e --no-cpu --no-configs > gpurun_out/r02_bench_fit2.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/r02_bench_fit2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fit'])"
