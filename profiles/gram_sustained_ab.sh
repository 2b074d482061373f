#!/bin/bash
# sustained config-3 Gram (40 back-to-back launches per process, 10 s apart): FP64 hybrid vs all-DMMA vs int8 tcgen05
run() { timeout 300 python - "$1" <<'PY'
import sys, json, torch
sys.path.insert(0, ".")
import paper_1604_04997_b200 as kc
N, F = 100_000_000, 40
X = torch.rand((N, F), dtype=torch.float64, device="cuda").mul_(9999.0).add_(1.0)
ts = []
for i in range(41):
    st = kc.GramStats.zeros(F, "cuda")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); kc.gram_accumulate(X, st, sliced=sys.argv[1] == "sliced"); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts = ts[1:]
print(sys.argv[1], json.dumps({"first5_ms": round(sum(ts[:5]) / 5, 3), "last20_ms": round(sum(ts[-20:]) / 20, 3)}))
PY
}
for r in 1 2; do
  sleep 10; run hybrid
  sleep 10; KCG_GRAM_HYBRID=0 run dmma
  sleep 10; run sliced
done
