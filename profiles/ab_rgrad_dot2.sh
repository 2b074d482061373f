#!/bin/bash
# A/B: refinement-gradient residual as a compensated dot product (new) vs double-double subtraction (old)
rm -rf /tmp/kcg_jit_cache-*
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_capi.py tests/test_dist_gpu.py tests/test_campaign.py tests/test_ref_dropin.py -q -m gpu -k "fit or refine or exact or grad or csv or campaign or dropin" 2>&1 | tail -2
for r in 1 2; do
  for v in old new; do
    echo -n "$v "; KCG_LIB=paper_1604_04997_b200/_lib/ab/libkcg_$v.so timeout 300 python profiles/time_fit5.py 1000 | tail -1
  done
done
