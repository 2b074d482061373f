nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/rc profiles/racecheck_mbarrier_probe.cu
for m in 0 1 2; do compute-sanitizer --tool racecheck /tmp/rc $m 2>&1 | grep -E "mode|SUMMARY|Error: Race" | head -3; done
