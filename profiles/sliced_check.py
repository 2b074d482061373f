"""Integer-sliced tcgen05 Gram (gram_sliced.cu) vs the FP64 path: parity on
awkward inputs and CUDA-event timing at config 3 (1e8 x 40).

    KCG_GRAM_SLICED=1 python profiles/sliced_check.py [check|time] [N] [F,...]

Parity compares G, X^T 1, colmax with an exact-as-possible fp64 reference
(torch matmul in fp64 on the same rows; the error is reported relative to
sum_r |x_ri| |x_rj|, the scale of fp64's own error bound)."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1604_04997_b200 as kc  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "check"
dev = "cuda"


def ref_stats(X):
    Xd = X.double()
    G = Xd.T @ Xd
    A = Xd.abs()
    scale = A.T @ A
    return G, Xd.sum(0), A.max(0).values, scale, A.sum(0)


def compare(X, tag):
    st = kc.gram_accumulate(X)
    G, x1, cm, scale, ascale = ref_stats(X)
    eg = float(((st.G - G).abs() / scale.clamp_min(1e-300)).max())
    ex = float(((st.xt1 - x1).abs() / ascale.clamp_min(1e-300)).max())
    cm_ok = bool(torch.equal(st.colmax, cm))
    sym = bool(torch.equal(st.G, st.G.T))
    return {"case": tag, "rows": X.shape[0], "F": X.shape[1], "G_err_rel_to_abs_scale": eg,
            "xt1_err_rel": ex, "colmax_exact": cm_ok, "symmetric": sym,
            "ok": eg < 1e-13 and ex < 1e-13 and cm_ok}


if mode == "check":
    g = torch.Generator(device=dev).manual_seed(7)
    res = []
    for F in [17, 20, 24, 25, 31, 32, 33, 36, 39, 40]:
        for n in [1, 127, 128, 129, 1000, 128 * 148 * 3 + 77, 128 * 300 * 148 + 5]:
            X = torch.rand((n, F), dtype=torch.float64, device=dev, generator=g).mul_(9999.0).add_(1.0)
            res.append(compare(X, "uniform"))
    F = 40
    n = 128 * 148 * 600 + 33  # > 2 segments per CTA
    # signed, wide dynamic range per column, zero columns, rising magnitudes (forces segment flushes)
    X = torch.randn((n, F), dtype=torch.float64, device=dev, generator=g)
    X[:, 3] = 0.0
    X[:, 5] *= torch.logspace(-30, 30, n, dtype=torch.float64, device=dev)
    X[:, 7] *= torch.exp2(torch.randint(-40, 40, (n,), device=dev, generator=g).double())
    X[:, 9] = torch.exp2(torch.randint(-5, 5, (n,), device=dev, generator=g).double())  # powers of two
    X[:, 11] = -X[:, 11].abs() * 1e140
    X[:, 12] = X[:, 12] * 1e-140
    res.append(compare(X, "signed/wide-range/zero/rising"))
    X = torch.randn((n, 33), dtype=torch.float64, device=dev, generator=g)
    X *= torch.linspace(1, 1e6, n, dtype=torch.float64, device=dev)[:, None]
    res.append(compare(X, "rising rows F=33"))
    # accumulate into existing stats
    X = torch.rand((200_000, 40), dtype=torch.float64, device=dev, generator=g)
    st = kc.gram_accumulate(X[:100_000])
    kc.gram_accumulate(X[100_000:], st)
    G = X.T @ X
    res.append({"case": "two calls", "G_err": float(((st.G - G).abs() / G.abs()).max()),
                "ok": float(((st.G - G).abs() / G.abs()).max()) < 1e-13})
    # non-finite
    X = torch.rand((50_000, 40), dtype=torch.float64, device=dev, generator=g)
    X[1234, 6] = float("inf")
    st = kc.gram_accumulate(X)
    res.append({"case": "inf", "G_nan_or_inf": bool((~torch.isfinite(st.G)).any()), "ok": bool((~torch.isfinite(st.G)).any())})
    bad = [r for r in res if not r["ok"]]
    print(json.dumps({"sliced": os.environ.get("KCG_GRAM_SLICED"), "cases": len(res), "failed": bad,
                      "worst_G": max(r.get("G_err_rel_to_abs_scale", 0) for r in res),
                      "worst_xt1": max(r.get("xt1_err_rel", 0) for r in res)}, indent=1))
    sys.exit(1 if bad else 0)

N = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000_000
out = {"sliced": os.environ.get("KCG_GRAM_SLICED")}
for F in [int(f) for f in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["40"])]:
    gen = torch.Generator(device=dev).manual_seed(4242)
    X = torch.rand((N, F), dtype=torch.float64, device=dev, generator=gen).mul_(9999.0).add_(1.0)
    st = kc.GramStats.zeros(F, X.device)
    for _ in range(3):
        kc.gram_accumulate(X, st)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        st = kc.GramStats.zeros(F, X.device)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        kc.gram_accumulate(X, st)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    Xs = X[:2_000_000]
    s2 = kc.gram_accumulate(Xs)
    ref = Xs.T @ Xs
    out[F] = {"ms": sorted(ts)[len(ts) // 2], "ms_min": min(ts), "GBps": 8.0 * F * N / min(ts) / 1e6,
              "rel_err_slice": float(((s2.G - ref).abs() / ref.abs()).max())}
    del X
print(json.dumps(out))
