#!/bin/bash
# End-of-round evidence: full GPU suite, memcheck, bench line, launch list,
# ncu --set full of the headline eval kernel and of the grid kernel.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tests/sanitize_smoke.py > gpurun_out/memcheck.log 2>&1; echo memcheck_rc=$?; tail -2 gpurun_out/memcheck.log
python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench_default.log > gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
  --log-file gpurun_out/launches_raw.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-fit > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:_tma --launch-skip 1 --launch-count 1 \
  -o gpurun_out/r01_eval_tma -f python profiles/profile_kernels.py eval > gpurun_out/ncu_eval.log 2>&1; echo ncu_eval=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:_grid --launch-skip 1 --launch-count 1 -o gpurun_out/r01_eval_grid -f python -c "
import sys; sys.path.insert(0, 'oracle')
import kc_oracle as ko, paper_1604_04997_b200 as kc, torch
a = ko.simdev_reference_alpha(); w = kc.ModelWeights(alpha=a, covered=[x != 0 for x in a])
p = kc.load_program('matmul_tiled_g16x16')
g = kc.Grid.for_program(p, {'n': (336, 336, 400), 'm': (336, 336, 400), 'l': (336, 336, 420)})
kc.predict_grid(w, p, g); kc.predict_grid(w, p, g); torch.cuda.synchronize()
" > gpurun_out/ncu_grid.log 2>&1; echo ncu_grid=$?
