# e2e leg: kcg_eval_predict_host, per-program D2H copies vs one 2D copy per chunk (KCG_HOST_2D)
for i in 1 2; do
  for e in "KCG_HOST_2D=0" "KCG_HOST_2D=1"; do
    env $e python bench.py --no-fit --no-cpu --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['e2e']; print('$e', round(d['value']/1e9,3), round(d['ms_per_step'],1), round(d['pcie_d2h_GBps_measured'],1), round(d['d2h_frac_of_measured'],3), 'pageable', round(d['pageable']['value']/1e9,3), d['pageable']['bitwise_equal_to_pinned'])"
  done
done
KCG_HOST_2D=1 python -m pytest tests/test_host_io.py -m gpu -q 2>&1 | tail -1
