#!/bin/bash
# A/B: column maxima with a warp-vote rare path (new) vs a select per value (old), materialised Gram
for r in 1 2 3; do
  for v in old new; do
    echo -n "$v "; KCG_LIB=paper_1604_04997_b200/_lib/ab/libkcg_$v.so timeout 300 python profiles/time_gram.py 100000000 40,36,48,24 | tail -1
  done
done
