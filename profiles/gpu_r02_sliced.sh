#!/bin/bash
# Integer-sliced tcgen05 Gram: parity (awkward inputs) + config-3 timing A/B vs the FP64 path.
mkdir -p gpurun_out
KCG_GRAM_SLICED=1 timeout 300 python profiles/sliced_check.py check > gpurun_out/sliced_check.log 2>&1; echo check_rc=$?
tail -8 gpurun_out/sliced_check.log
for r in 1 2; do
  KCG_GRAM_SLICED=1 timeout 300 python profiles/sliced_check.py time 100000000 40,33,32,24 2>&1 | tail -1
  timeout 300 python profiles/sliced_check.py time 100000000 40,33,32,24 2>&1 | tail -1
done
KCG_GRAM_SLICED=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:kcg_gram_sliced --launch-skip 2 --launch-count 1 -o gpurun_out/r02_gram_sliced -f python profiles/time_gram.py 8000000 40 > gpurun_out/ncu_sliced.log 2>&1; echo ncu=$?
