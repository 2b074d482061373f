#!/bin/bash
# predict folding + argmin variants: full parity suite, then argmin A/B
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t4.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/t4.log
for c in 0 3 4; do KCG_ARGMIN_CTAS=$c python profiles/time_argmin.py; done
python bench.py --no-e2e --no-cpu --no-fit --extras --steps 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['extras']
print('headline', d['value'], d['roofline']['frac']); print('argmin', e['config4_argmin_fused']['ms']); print('grid', e['config4_grid_descriptor']['points_per_s'])"
