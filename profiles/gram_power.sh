#!/bin/bash
# config-3 Gram under sustained load: SM clock, power and throttle reasons sampled while 40 back-to-back Grams run
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_throttle_reasons.active --format=csv,noheader -lms 50 > gpurun_out/gram_power.csv &
P=$!
timeout 300 python - <<'PY'
import sys, json, torch
sys.path.insert(0, ".")
import paper_1604_04997_b200 as kc
N, F = 100_000_000, 40
X = torch.rand((N, F), dtype=torch.float64, device="cuda").mul_(9999.0).add_(1.0)
ts = []
for i in range(40):
    st = kc.GramStats.zeros(F, "cuda")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); kc.gram_accumulate(X, st); b.record(); torch.cuda.synchronize(); ts.append(round(a.elapsed_time(b), 3))
print(json.dumps({"gram_ms_sequence": ts}))
PY
kill $P
grep -v " 120 MHz" gpurun_out/gram_power.csv | head -40
