#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multi.py tests/test_host_io.py -m gpu -x -q > gpurun_out/r02_bulk_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r02_bulk_tests.log
python profiles/time_multi.py 551
KCG_MULTI_BULK=0 python profiles/time_multi.py 551
KCG_MULTI_OBUF=1 python profiles/time_multi.py 551
KCG_MULTI_BULK_CTAS=2 KCG_MULTI_OBUF=1 KCG_MULTI_BULK_RING_KB=48 python profiles/time_multi.py 551
KCG_MULTI_BULK_CTAS=2 KCG_MULTI_OBUF=2 KCG_MULTI_BULK_RING_KB=24 python profiles/time_multi.py 551
KCG_MULTI_BULK_RING_KB=120 python profiles/time_multi.py 551
