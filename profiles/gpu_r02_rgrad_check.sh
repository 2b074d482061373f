#!/bin/bash
# refinement-gradient defaults (64-register cap, strided rows, resident grid): fit parity tests + timing
rm -rf /tmp/kcg_jit_cache-*
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_capi.py tests/test_dist_gpu.py tests/test_campaign.py tests/test_ref_dropin.py tests/test_fuzz.py -q -m gpu 2>&1 | tail -2
timeout 300 python profiles/time_fit5.py 1000 | tail -1
