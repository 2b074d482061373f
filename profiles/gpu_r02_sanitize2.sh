#!/bin/bash
# compute-sanitizer over the Gram and one-pass kernels: memcheck / synccheck at sizes where the TMA
# rings refill, racecheck at one wave (it cannot see the fence-and-counter hand-back); GPU tests; A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_tests_ring.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/r02_tests_ring.log
for t in sanitize_gram sanitize_multi; do
  for tool in memcheck synccheck; do
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tests/$t.py > gpurun_out/r02_${t}_$tool.log 2>&1; echo $t $tool=$?; grep -E "SUMMARY" gpurun_out/r02_${t}_$tool.log | tail -1
  done
  KCG_SANITIZE_SMALL=1 timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tests/$t.py > gpurun_out/r02_${t}_racecheck.log 2>&1; echo $t racecheck=$?; grep -E "SUMMARY" gpurun_out/r02_${t}_racecheck.log | tail -1
done
for i in 1 2; do
  python profiles/time_gram.py 100000000 9,18,24,32,40,48,56,80 | sed 's/^/new /'
  KCG_LIB=_ab/libkcg_prev.so python profiles/time_gram.py 100000000 9,18,24,32,40,48,56,80 | sed 's/^/old /'
done
python profiles/time_multi.py 2>/dev/null | tail -1 | sed 's/^/new /'
KCG_LIB=_ab/libkcg_prev.so python profiles/time_multi.py 2>/dev/null | tail -1 | sed 's/^/old /'
