#!/bin/bash
# refinement-gradient kernel alone: CTAs per SM (register cap) x row order
for r in 1 2; do
for cfg in "3 0" "2 0" "2 1" "4 0" "4 1" "1 0"; do
  set -- $cfg
  echo -n "rgrad_ctas=$1 strided=$2 "; KCG_RGRAD_CTAS=$1 KCG_RGRAD_STRIDED=$2 timeout 300 python profiles/time_fit5.py 1000 | tail -1
done
done
