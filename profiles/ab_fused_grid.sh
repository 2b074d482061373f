#!/bin/bash
# fused Gram / residual grid at the resident CTA count vs the register-cap target; rgrad defaults
for r in 1 2 3; do
  for v in 0 1; do echo -n "resident=$v "; KCG_FUSED_GRID_RESIDENT=$v timeout 300 python profiles/time_fit5.py 1000 | tail -1; done
done
