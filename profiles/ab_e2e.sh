# A/B of the end-to-end leg's chunking (KCG_E2E_CHUNK sizes, KCG_E2E_STREAMS)
for e in "KCG_E2E_CHUNK=4194304 KCG_E2E_STREAMS=3" "KCG_E2E_CHUNK=1048576 KCG_E2E_STREAMS=4" "KCG_E2E_CHUNK=16777216 KCG_E2E_STREAMS=3" "KCG_E2E_CHUNK=8388608 KCG_E2E_STREAMS=2" "KCG_E2E_CHUNK=2097152 KCG_E2E_STREAMS=6"; do
  env $e python bench.py --no-fit --no-cpu --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['e2e']; print('$e', round(d['value']/1e9,3), round(d['ms_per_step'],1), round(d['pcie_d2h_GBps_measured'],1), round(d['d2h_frac_of_measured'],3))"
done
