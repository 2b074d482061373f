#!/bin/bash
# refinement gradient: register cap (KCG_RGRAD_CTAS) x grid CTAs per SM (KCG_RGRAD_GRID, 0 = resident count) x row order
for r in 1 2; do
for cfg in "3 0 0" "2 0 1" "4 0 1" "4 4 1" "4 2 1" "3 2 1" "4 0 0"; do
  set -- $cfg
  echo -n "regcap_ctas=$1 grid=$2 strided=$3 "; KCG_RGRAD_CTAS=$1 KCG_RGRAD_GRID=$2 KCG_RGRAD_STRIDED=$3 timeout 300 python profiles/time_fit5.py 1000 | tail -1
done
done
