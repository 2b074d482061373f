#!/bin/bash
timeout 600 python -m pytest tests/test_multi.py -m gpu -x -q 2>&1 | tail -1
KCG_MULTI_BULK_CTA=1 timeout 600 python -m pytest tests/test_multi.py -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do KCG_MULTI_BULK=0 python profiles/time_multi.py 551; done
for i in 1 2; do python profiles/time_multi.py 551; done
for c in 2 3; do for i in 1 2; do KCG_MULTI_BULK_CTA=1 KCG_MULTI_BULK_CTAS=$c python profiles/time_multi.py 551; done; done
KCG_MULTI_BULK_CTA=1 KCG_MULTI_BULK_CTAS=2 KCG_MULTI_BULK_RING_KB=72 python profiles/time_multi.py 551
