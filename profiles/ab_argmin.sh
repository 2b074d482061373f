#!/bin/bash
# same-box A/B of the argmin kernel: _ab_old (a previous commit's tree, with
# its own profiles/time_argmin.py so that it imports its own package) vs the tree
for r in 1 2; do
  (cd _ab_old && python profiles/time_argmin.py) | sed 's/^/old /'
  python profiles/time_argmin.py | sed 's/^/new /'
done
