#!/bin/bash
# A/B of the sliced Gram's input path: L2 bulk prefetch distance and load flavour (1e8 x 40)
for r in 1 2; do
for cfg in "6 0" "0 0" "12 0" "6 1" "0 1"; do
  set -- $cfg
  echo -n "pf=$1 ldg=$2 "; KCG_GRAM_SLICED=1 KCG_SLICED_PF=$1 KCG_SLICED_LDG=$2 timeout 300 python profiles/sliced_check.py time 100000000 40 | tail -1
done
done
