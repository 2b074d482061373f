#!/bin/bash
# refinement gradient: rows in flight per thread (unroll) x register cap
for r in 1 2; do
for cfg in "4 1" "4 2" "4 4" "3 2" "2 2" "2 4"; do
  set -- $cfg
  echo -n "ctas=$1 unroll=$2 "; KCG_RGRAD_CTAS=$1 KCG_RGRAD_UNROLL=$2 timeout 300 python profiles/time_fit5.py 1000 | tail -1
done
done
