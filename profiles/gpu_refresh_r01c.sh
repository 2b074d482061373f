#!/bin/bash
# Evidence refresh after a kernel change: memcheck, bench line, launch list,
# ncu --set full of the headline eval, argmin and fused Gram kernels.
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tests/sanitize_smoke.py > gpurun_out/memcheck.log 2>&1; echo memcheck_rc=$?; tail -1 gpurun_out/memcheck.log
python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench_default.log > gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
  --log-file gpurun_out/launches_raw.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-fit > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:_tma --launch-skip 1 --launch-count 1 \
  -o gpurun_out/r01_eval_tma -f python profiles/profile_kernels.py eval > gpurun_out/ncu_eval.log 2>&1; echo ncu_eval=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:argmin --launch-skip 1 --launch-count 1 \
  -o gpurun_out/r01_argmin -f python profiles/profile_kernels.py argmin > gpurun_out/ncu_argmin.log 2>&1; echo ncu_argmin=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_gram_matmul --launch-skip 1 --launch-count 1 \
  -o gpurun_out/r01_gram_fused -f python profiles/profile_kernels.py gram_fused > gpurun_out/ncu_gram_fused.log 2>&1; echo ncu_gram_fused=$?
