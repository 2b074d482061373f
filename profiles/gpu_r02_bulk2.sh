#!/bin/bash
for i in 1 2; do KCG_MULTI_BULK=0 python profiles/time_multi.py 551; done
for i in 1 2; do KCG_MULTI_BULK_CTAS=2 KCG_MULTI_OBUF=1 KCG_MULTI_BULK_RING_KB=48 python profiles/time_multi.py 551; done
KCG_MULTI_BULK_CTAS=2 KCG_MULTI_OBUF=1 KCG_MULTI_BULK_RING_KB=64 python profiles/time_multi.py 551
KCG_MULTI_BULK_CTAS=2 KCG_MULTI_OBUF=2 KCG_MULTI_BULK_RING_KB=16 python profiles/time_multi.py 551
KCG_MULTI_BULK_CTAS=3 KCG_MULTI_OBUF=1 KCG_MULTI_BULK_RING_KB=16 python profiles/time_multi.py 551
