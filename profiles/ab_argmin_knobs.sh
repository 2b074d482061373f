# A/B of the argmin kernel's knobs on one box (KCG_ARGMIN_*)
for r in 1 2; do
  for e in "KCG_ARGMIN_PAIR=0" "KCG_ARGMIN_PAIR=1" "KCG_ARGMIN_PAIR=1 KCG_ARGMIN_CTAS=3" "KCG_ARGMIN_PAIR=1 KCG_ARGMIN_CTAS=2"; do
    env $e python profiles/time_argmin.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['ms'],3), d['hist'])"
  done
done
KCG_ARGMIN_PAIR=1 python -m pytest tests -m gpu -q -k "argmin" 2>&1 | tail -1
