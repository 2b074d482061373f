#!/bin/bash
# DMMA Gram stage hand-back: release before / after the last k-step, against the bare-counter build (_ab/libkcg_prev.so)
for i in 1 2; do
  python profiles/time_gram.py 100000000 24,32,48,56 | sed 's/^/new /'
  KCG_DMMA_LATE_RELEASE=1 python profiles/time_gram.py 100000000 24,32,48,56 | sed 's/^/late /'
  KCG_LIB=_ab/libkcg_prev.so python profiles/time_gram.py 100000000 24,32,48,56 | sed 's/^/old /'
done
