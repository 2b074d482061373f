#!/bin/bash
# refinement gradient: pairwise-tree compensated sum (new) vs sequential Dot2 (old); fit tests on the new one
rm -rf /tmp/kcg_jit_cache-*
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_refined_objective.py tests/test_campaign.py tests/test_dist_gpu.py tests/test_ref_dropin.py -q -m gpu -k "fit or refine or exact or grad or csv or campaign or dropin or refined or objective or rank" 2>&1 | tail -2
for r in 1 2 3; do
  for v in old new; do
    echo -n "$v "; KCG_LIB=paper_1604_04997_b200/_lib/ab/libkcg_$v.so timeout 300 python profiles/time_fit5.py 1000 | tail -1
  done
done
