#!/bin/bash
# Round-1 GPU evidence run 2: grid/columns tests, Gram DMMA timing, grid timing,
# ncu of the argmin and of a large enumeration walk.
mkdir -p gpurun_out
python -m pytest tests/test_grid.py tests/test_gpu_parity.py -m gpu -q -k "grid or columns or gram or fit" > gpurun_out/t2.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t2.log
python profiles/time_gram.py 100000000 40,24,9 2>&1 | tail -1
python bench.py --no-e2e --no-cpu --no-fit --extras --steps 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['extras']
print('headline', d['value'], d['roofline']['frac']); print('argmin', e['config4_argmin_fused']['ms']); print('grid', e['config4_grid_descriptor']); print('gram', e['config3_gram_1e8x40']['ms'], e['config3_gram_1e8x40']['hbm_frac'])"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kcg_argmin --launch-skip 1 --launch-count 1 -o gpurun_out/r01_argmin -f python profiles/profile_kernels.py argmin > gpurun_out/ncu_argmin.log 2>&1; echo ncu_argmin=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kcg_enum_walk --launch-skip 7 --launch-count 1 -o gpurun_out/r01_enum_walk -f python -c "
import paper_1604_04997_b200 as kc
p = kc.load_enum_program('fd_stencil_g16x16')
p.enumerate_points({'n': 1024}); p.enumerate_points({'n': 8192})
" > gpurun_out/ncu_enum.log 2>&1; echo ncu_enum=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kcg_gram_dmma --launch-skip 1 --launch-count 1 -o gpurun_out/r01_gram_dmma -f python profiles/profile_kernels.py gram > gpurun_out/ncu_gram.log 2>&1; echo ncu_gram=$?
