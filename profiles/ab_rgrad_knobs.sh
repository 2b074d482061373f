#!/bin/bash
# rgrad / residual occupancy and unroll knobs (they also move the fused Gram)
for cfg in "3 1 0" "4 1 0" "2 1 0" "3 2 0" "3 4 0" "3 1 1" "4 2 0"; do
  set -- $cfg
  echo -n "ctas=$1 unroll=$2 strided=$3 "; KCG_FUSED_CTAS=$1 KCG_FUSED_UNROLL=$2 KCG_FUSED_STRIDED=$3 timeout 300 python profiles/time_fit5.py 1000 | tail -1
done
