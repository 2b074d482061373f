# A/B of the argmin kernel's knobs on one box (KCG_ARGMIN_*). Results quoted
# in DESIGN.md; a two-sizes-per-thread variant measured 3.57 ms against 3.35
# and was removed.
for r in 1 2; do
  for e in "KCG_ARGMIN_PREFETCH=0" "KCG_ARGMIN_PREFETCH=1" "KCG_ARGMIN_PREFETCH=1 KCG_ARGMIN_CTAS=3" "KCG_ARGMIN_PREFETCH=1 KCG_ARGMIN_CTAS=4"; do
    env $e python profiles/time_argmin.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['ms'],3), d['hist'])"
  done
done
