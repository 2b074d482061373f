# A/B: 64- vs 128-row tiles of the row-split DMMA Gram for 4-5 column blocks
for e in "KCG_DMMA_TALL=0" "KCG_DMMA_TALL=1"; do
  echo "$e $(env $e python profiles/time_gram.py 100000000 25,32,33,40)"
done
