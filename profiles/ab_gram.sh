# A/B: grouped row-split DMMA Gram (KCG_WIDE_GROUPED=1) vs the per-warp-run kernel for F > 72
for e in "KCG_WIDE_GROUPED=0" "KCG_WIDE_GROUPED=1"; do
  echo "$e $(env $e python profiles/time_gram.py 20000000 80,96,111,149,160)"
done
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gram" 2>&1 | tail -1
timeout 300 compute-sanitizer --tool memcheck --print-limit 10 python tests/sanitize_gram.py 2>&1 | tail -1
timeout 300 compute-sanitizer --tool racecheck --print-limit 10 python tests/sanitize_gram.py 2>&1 | tail -1
