#!/bin/bash
# ncu --set full of the integer-sliced tcgen05 Gram (8e6 x 40 rows)
mkdir -p gpurun_out
KCG_GRAM_SLICED=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_gram_sliced --launch-skip 2 --launch-count 1 -o gpurun_out/r02_gram_sliced -f python profiles/time_gram.py 8000000 40 > gpurun_out/ncu_sliced.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_sliced.log
