#!/bin/bash
# objective from the refinement pass: its tests, the fit / dist tests, config-5 timing in the bench
rm -rf /tmp/kcg_jit_cache-*
timeout 1500 python -m pytest tests/test_refined_objective.py tests/test_dist_gpu.py tests/test_gpu_parity.py -q -m gpu -k "refined or fit or objective or rank" 2>&1 | tail -3
timeout 900 python bench.py --no-e2e --no-cpu --no-configs > gpurun_out/r02_bench_refobj.log 2>&1; echo bench=$?
tail -1 gpurun_out/r02_bench_refobj.log > gpurun_out/r02_bench_refobj.json
