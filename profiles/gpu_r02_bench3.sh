#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multi.py tests/test_host_io.py tests/test_dist_gpu.py -m gpu -x -q 2>&1 | tail -1
python profiles/time_multi.py 551 --stream
timeout 900 python bench.py > gpurun_out/r02_bench3.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/r02_bench3.log > gpurun_out/r02_bench3.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches_raw3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-fit --no-configs > gpurun_out/r02_ncu_list3.log 2>&1; echo ncu_list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kcg_multi_v6_tmab --launch-skip 2 --launch-count 1 \
  -o gpurun_out/r02_multi_bulk -f python profiles/time_multi.py 551 > gpurun_out/r02_ncu_bulk.log 2>&1; echo ncu_full=$?
