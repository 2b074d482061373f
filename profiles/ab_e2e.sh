# A/B of kcg_eval_predict_host's chunking (KCG_HOST_CHUNK points, KCG_HOST_STREAMS) in the e2e leg
for e in "KCG_HOST_CHUNK=4194304 KCG_HOST_STREAMS=3" "KCG_HOST_CHUNK=8388608 KCG_HOST_STREAMS=2" "KCG_HOST_CHUNK=2097152 KCG_HOST_STREAMS=4" "KCG_HOST_CHUNK=4194304 KCG_HOST_STREAMS=3"; do
  env $e python bench.py --no-fit --no-cpu --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['e2e']; print('$e', round(d['value']/1e9,3), round(d['ms_per_step'],1), round(d['pcie_d2h_GBps_measured'],1), round(d['d2h_frac_of_measured'],3), 'pageable', round(d['pageable']['value']/1e9,3), d['pageable']['bitwise_equal_to_pinned'])"
done
