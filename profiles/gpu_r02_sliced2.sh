#!/bin/bash
# Integer-sliced tcgen05 Gram: the GPU parity test + config-3 timing A/B vs the FP64 hybrid.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gram_sliced.py -q -m gpu 2>&1 | tail -3
for r in 1 2; do
  KCG_GRAM_SLICED=1 timeout 300 python profiles/sliced_check.py time 100000000 40,32,24 2>&1 | tail -1
  timeout 300 python profiles/sliced_check.py time 100000000 40,32,24 2>&1 | tail -1
done
