#!/bin/bash
# GPU tests with the host code under AddressSanitizer + UBSan (the CUDA
# kernels are the regular build; protect_shadow_gap=0 lets the CUDA driver map)
make -C paper_1604_04997_b200/csrc asan > /dev/null 2>&1 || echo "asan build failed"
export LD_PRELOAD="$(/usr/bin/g++ -print-file-name=libasan.so) $(/usr/bin/g++ -print-file-name=libstdc++.so)"
export ASAN_OPTIONS=detect_leaks=0:protect_shadow_gap=0 KCG_LIB=paper_1604_04997_b200/_lib/asan/libkcg.so
timeout 2400 python -m pytest tests/test_multi.py tests/test_host_io.py tests/test_enumerate.py tests/test_grid.py tests/test_capi.py tests/test_campaign.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_asan_gpu.log 2>&1; echo rc=$?
grep -E "==ERROR|runtime error|passed|failed" gpurun_out/r02_asan_gpu.log | head
