#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_tests_all.log 2>&1; echo tests_rc=$?; tail -8 gpurun_out/r02_tests_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/r02_smoke.log
