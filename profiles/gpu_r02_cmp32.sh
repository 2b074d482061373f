#!/bin/bash
timeout 1200 python -m pytest tests/test_fuzz.py tests/test_multi.py tests/test_gpu_parity.py tests/test_grid.py -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do python profiles/time_argmin.py; done
for i in 1 2; do python profiles/time_multi.py 551; done
