#!/bin/bash
# int8 tcgen05 Gram: 7 digits (56-bit) vs 6 digits (48-bit, 27% fewer operand bytes per tile)
KCG_GRAM_SLICED=1 KCG_SLICED_DIGITS=6 timeout 300 python profiles/sliced_check.py check 2>&1 | grep -E '"failed"|worst' | head -3
for r in 1 2; do
  for d in 7 6; do echo -n "digits=$d "; KCG_GRAM_SLICED=1 KCG_SLICED_DIGITS=$d timeout 300 python profiles/sliced_check.py time 100000000 40 | tail -1; done
done
