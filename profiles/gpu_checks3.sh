#!/bin/bash
# argmin (TMA ring, weights by value) + odd-width DMMA Gram: parity and timing
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "argmin or gram_accumulate or fit" > gpurun_out/t3.log 2>&1; echo tests_rc=$?; tail -15 gpurun_out/t3.log
python profiles/time_gram.py 100000000 40,9,47 2>&1 | tail -1
python bench.py --no-e2e --no-cpu --no-fit --extras --steps 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['extras']
print('headline', d['value'], d['roofline']['frac']); print('argmin', e['config4_argmin_fused']); print('grid', e['config4_grid_descriptor']['points_per_s'])"
