# A/B of the row-split DMMA Gram at one vs two CTAs per SM (KCG_DMMA_ONE_CTA_NB = first NB at one CTA)
for e in "KCG_DMMA_ONE_CTA_NB=9" "KCG_DMMA_ONE_CTA_NB=1" "KCG_DMMA_ONE_CTA_NB=6"; do
  echo "$e $(env $e python profiles/time_gram.py 100000000 9,16,24,32,40,48)"
done
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gram" 2>&1 | tail -1
