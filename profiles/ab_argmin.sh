#!/bin/bash
# same-box A/B of the argmin kernel: _ab_old (previous commit) vs the tree
for r in 1 2; do
  (cd _ab_old && PYTHONPATH=. python ../profiles/time_argmin.py) | sed 's/^/old /'
  python profiles/time_argmin.py | sed 's/^/new /'
done
