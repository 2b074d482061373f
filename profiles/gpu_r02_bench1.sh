#!/bin/bash
# Round 2: the one-pass headline on the GPU -- tests, bench line, ncu evidence.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multi.py tests/test_host_io.py tests/test_capi.py -m gpu -x -q > gpurun_out/r02_tests_b1.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r02_tests_b1.log
timeout 900 python bench.py > gpurun_out/r02_bench_b1.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/r02_bench_b1.log > gpurun_out/r02_bench_b1.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches_raw.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-fit --no-configs > gpurun_out/r02_ncu_list.log 2>&1; echo ncu_list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kcg_multi_v6_tma --launch-skip 2 --launch-count 1 \
  -o gpurun_out/r02_multi_full -f python profiles/time_multi.py 551 > gpurun_out/r02_ncu_full.log 2>&1; echo ncu_full=$?
