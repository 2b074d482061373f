# A/B: row-split DMMA (KCG_DMMA_MAXF covers it) vs the grouped wide kernel for 49 <= F <= 72
for e in "KCG_DMMA_MAXF=72" "KCG_DMMA_MAXF=64" "KCG_DMMA_MAXF=48"; do
  echo "$e $(env $e python profiles/time_gram.py 50000000 52,56,64,66,72)"
done
