# A/B of the register-path fused Gram / residual knobs (KCG_FUSED_*), 2^28 config-5 rows
for i in 1 2; do
  for e in "KCG_FUSED_UNROLL=1" "KCG_FUSED_UNROLL=4" "KCG_FUSED_STRIDED=1" "KCG_FUSED_STRIDED=1 KCG_FUSED_UNROLL=4" "KCG_FUSED_STRIDED=1 KCG_FUSED_UNROLL=2"; do
    echo "$e $(env $e python profiles/time_fused.py)"
  done
done
KCG_FUSED_STRIDED=1 KCG_FUSED_UNROLL=4 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "fused or fit" 2>&1 | tail -1
