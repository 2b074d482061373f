#!/bin/bash
mkdir -p gpurun_out
KCG_MULTI_CTAS=1 KCG_MULTI_PREFETCH=0 python profiles/time_multi.py 551 --stream
KCG_MULTI_CTAS=2 KCG_MULTI_PREFETCH=0 KCG_MULTI_RING_KB=48 python profiles/time_multi.py
KCG_MULTI_CTAS=1 KCG_MULTI_PREFETCH=0 KCG_MULTI_RING_KB=48 python profiles/time_multi.py
KCG_MULTI_CTAS=1 KCG_MULTI_PREFETCH=0 KCG_MULTI_RING_KB=72 python profiles/time_multi.py
