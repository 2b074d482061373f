#!/bin/bash
# Round-end evidence: full GPU suite, memcheck, extras bench line, ncu of the
# grouped wide Gram (F = 149) and of the row-split Gram (F = 40, 128-row tiles).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/gpu_tests.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tests/sanitize_smoke.py > gpurun_out/memcheck.log 2>&1; echo memcheck_rc=$?; tail -1 gpurun_out/memcheck.log
python bench.py --extras > gpurun_out/bench_extras.log 2>&1; echo extras_rc=$?; tail -1 gpurun_out/bench_extras.log > gpurun_out/bench_extras.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_group --launch-skip 1 --launch-count 1 -o gpurun_out/r01_gram_group -f python -c "
import torch, paper_1604_04997_b200 as kc
X = torch.rand((1 << 21, 149), dtype=torch.float64, device='cuda')
kc.gram_accumulate(X); kc.gram_accumulate(X); torch.cuda.synchronize()
" > gpurun_out/ncu_group.log 2>&1; echo ncu_group=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_dmma --launch-skip 1 --launch-count 1 \
  -o gpurun_out/r01_gram_dmma -f python profiles/profile_kernels.py gram > gpurun_out/ncu_gram.log 2>&1; echo ncu_gram=$?
