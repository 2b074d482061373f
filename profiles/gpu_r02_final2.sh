#!/bin/bash
# End-of-round evidence: fresh-cache bench, the full GPU suite, smoke, the Gram sanitizer target run plainly
mkdir -p gpurun_out
rm -rf /tmp/kcg_jit_cache-* /tmp/kcg_jit_cache
s=$(date +%s); timeout 1200 python bench.py > gpurun_out/r02_bench_final2.log 2>&1; echo bench_rc=$? wall_s=$(( $(date +%s) - s ))
tail -1 gpurun_out/r02_bench_final2.log > gpurun_out/r02_bench_final2.json
s=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02_tests_final2.log 2>&1; echo tests_rc=$? wall_s=$(( $(date +%s) - s )); tail -2 gpurun_out/r02_tests_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python tests/sanitize_gram.py 2>&1 | tail -1
