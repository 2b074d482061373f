#!/bin/bash
# hybrid Gram tile height per warp group, interleaved with the all-DMMA kernel
for i in 1 2; do
for r in 96 144; do KCG_GRAM_HYBRID_R=$r python profiles/time_gram.py 100000000 40 | sed "s/^/R=$r /"; done
KCG_GRAM_HYBRID=0 python profiles/time_gram.py 100000000 40 | sed "s/^/dmma /"
for r in 64 128; do KCG_GRAM_HYBRID=1 KCG_GRAM_HYBRID_R4=$r python profiles/time_gram.py 100000000 32,36 | sed "s/^/all R4=$r /"; done
KCG_GRAM_HYBRID=0 python profiles/time_gram.py 100000000 32,36 | sed "s/^/dmma /"
done
