#!/bin/bash
# Round-1 GPU evidence run: full -m gpu suite, memcheck over every kernel family,
# ncu --set full of the enumeration walk and the grid evaluate kernel.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tests/sanitize_smoke.py > gpurun_out/memcheck.log 2>&1; echo memcheck_rc=$?; tail -4 gpurun_out/memcheck.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kcg_enum_walk --launch-skip 3 --launch-count 1 -o gpurun_out/r01_enum_walk -f python -c "
import paper_1604_04997_b200 as kc
p = kc.load_enum_program('fd_stencil_g16x16')
p.enumerate_points({'n': 1024}); p.enumerate_points({'n': 8192})
" > gpurun_out/ncu_enum.log 2>&1; echo ncu_enum=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:_grid --launch-skip 1 --launch-count 1 -o gpurun_out/r01_eval_grid -f python -c "
import sys; sys.path.insert(0, 'oracle')
import kc_oracle as ko, paper_1604_04997_b200 as kc, torch
a = ko.simdev_reference_alpha(); w = kc.ModelWeights(alpha=a, covered=[x != 0 for x in a])
p = kc.load_program('matmul_tiled_g16x16')
g = kc.Grid.for_program(p, {'n': (336, 336, 400), 'm': (336, 336, 400), 'l': (336, 336, 420)})
kc.predict_grid(w, p, g); kc.predict_grid(w, p, g); torch.cuda.synchronize()
" > gpurun_out/ncu_grid.log 2>&1; echo ncu_grid=$?
ls gpurun_out
