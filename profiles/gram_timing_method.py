"""Config-3 Gram: per-call CUDA-event timing (min / median of single launches)
against the bench's back-to-back mean with the statistics zeroed per call."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1604_04997_b200 as kc  # noqa: E402

N, F = 100_000_000, 40
g = torch.Generator(device="cuda").manual_seed(4242)
X = torch.rand((N, F), dtype=torch.float64, device="cuda", generator=g).mul_(9999.0).add_(1.0)
st = kc.GramStats.zeros(F, "cuda")
stream = torch.cuda.current_stream().cuda_stream


def c3():
    st.G.zero_(); st.xt1.zero_(); st.colmax.zero_()
    kc.api.check(kc.api.lib().kcg_gram_accumulate(X.data_ptr(), N, F, F, st.G.data_ptr(), st.xt1.data_ptr(),
                                                  st.colmax.data_ptr(), stream))


out = {}
for rep in range(3):
    for _ in range(2):
        c3()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        c3()
    b.record()
    torch.cuda.synchronize()
    out.setdefault("back_to_back_mean_ms", []).append(a.elapsed_time(b) / 5)
    ts = []
    for _ in range(5):
        a.record(); c3(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    out.setdefault("per_call_median_ms", []).append(sorted(ts)[2])
print(json.dumps(out))
