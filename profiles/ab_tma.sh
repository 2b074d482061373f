# A/B of the headline TMA kernel's knobs (KCG_TMA_*), default bench step only
run() { env "$@" python bench.py --no-fit --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']/1e9,1), round(d['roofline']['frac_of_same_mix'],4))"; }
for i in 1 2; do
  run KCG_TMA_TILE_Q=4
  run KCG_TMA_TILE_Q=3
  run KCG_TMA_TILE_Q=3 KCG_TMA_RING_KB=72
  run KCG_TMA_TILE_Q=5
done
