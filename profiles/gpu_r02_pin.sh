#!/bin/bash
mkdir -p gpurun_out
timeout 600 ./oracle/_ref/ref_dropin > gpurun_out/r02_ref_dropin.json 2> gpurun_out/r02_ref_dropin.err; echo dropin_rc=$?; cat gpurun_out/r02_ref_dropin.json; tail -3 gpurun_out/r02_ref_dropin.err
timeout 1500 python -m pytest tests/test_config2.py tests/test_ref_dropin.py tests/test_gpu_parity.py -m gpu -q -k "config2 or dropin or fused_reaches" --durations=10 > gpurun_out/r02_tests_pin.log 2>&1; echo tests_rc=$?; tail -18 gpurun_out/r02_tests_pin.log
