#!/bin/bash
# e2e leg (kcg_eval_predict_host, pinned): chunk size x stream count
for r in 1 2; do
for cfg in "4194304 3" "2097152 3" "1048576 3" "8388608 3" "2097152 4" "1048576 4" "4194304 2"; do
  set -- $cfg
  KCG_HOST_CHUNK=$1 KCG_HOST_STREAMS=$2 timeout 300 python bench.py --no-fit --no-cpu --no-configs --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['e2e']; print('chunk=$1 streams=$2', round(d['value']/1e9,3), round(d['ms_per_step'],1), round(d['d2h_frac_of_measured'],3))"
done
done
