#!/bin/bash
# sliced Gram through its C ABI: GPU tests, the default bench line (config 3 carries the int8 alternative), ncu of the kept kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gram_sliced.py -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r02_bench_sliced.log 2>&1; echo bench=$?; tail -1 gpurun_out/r02_bench_sliced.log > gpurun_out/r02_bench_sliced.json
KCG_GRAM_SLICED=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_gram_sliced --launch-skip 2 --launch-count 1 -o gpurun_out/r02_gram_sliced -f python profiles/time_gram.py 8000000 40 > gpurun_out/ncu_sliced.log 2>&1; echo ncu=$?
