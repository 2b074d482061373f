#!/bin/bash
# fit_from_csv with the objective from the last refinement pass: campaign / CSV / drop-in tests and the config-1 timing
rm -rf /tmp/kcg_jit_cache-*
timeout 1500 python -m pytest tests/test_campaign.py tests/test_gpu_parity.py tests/test_refined_objective.py -q -m gpu -k "csv or campaign or fit or refined or objective" 2>&1 | tail -2
timeout 900 python bench.py --no-e2e --no-cpu --no-fit > gpurun_out/r02_bench_csvfit.log 2>&1; echo bench=$?
tail -1 gpurun_out/r02_bench_csvfit.log > gpurun_out/r02_bench_csvfit.json
