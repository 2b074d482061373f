# A/B: row-split DMMA (one CTA/SM) vs the per-width kernel for 65 <= F <= 72 (KCG_DMMA_MAXF)
for e in "KCG_DMMA_MAXF=64" "KCG_DMMA_MAXF=72"; do
  echo "$e $(env $e python profiles/time_gram.py 50000000 66,72)"
done
KCG_DMMA_MAXF=72 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gram" 2>&1 | tail -1
