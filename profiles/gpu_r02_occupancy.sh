#!/bin/bash
# launch shape of every kernel in a short bench run: grid vs the CTAs/SM that registers and shared memory admit
mkdir -p gpurun_out
timeout 1200 ncu --metrics launch__grid_size,launch__block_size,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,gpu__time_duration.sum --csv -c 600 --log-file gpurun_out/r02_occupancy.csv python bench.py --steps 1 --warmup 3 --no-cpu --side 200 > gpurun_out/occ.log 2>&1; echo rc=$?
