"""BASELINE config 2 pinned end to end -> tests/golden/config2_hashes.json
(test infrastructure; needs oracle/_ref built from /root/reference).

Config 2 is 250,000 points per test kernel: skinny matmul
(16u, 128u, 16u), conv 16u, fd_stencil 16u, nbody 256u, u = 1..250000.
The reference evaluates every point (oracle/_ref/kcref_config2):
  * skinny and conv through the symbolic path (extract_properties once,
    evaluate_properties + predict per point) -- all 250,000 points;
  * fd_stencil and nbody are not symbolic in the reference: bound mode
    (extract_properties(k, b, cap 2e7), enumeration) for every u up to the
    last one the 2e7 enumeration cap admits.
Each point becomes F int128 counts (the GPU program's keys) + the fp64
prediction bits; the records are hashed (sha256) in blocks of 1000 points,
so tests/test_config2.py can compare every count and every prediction of
the GPU's 1e6 points without shipping 150 MB of fixtures.

    python tests/gen/gen_config2.py [--procs 8]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import hashlib
import json
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
EXE = ROOT / "oracle" / "_ref" / "kcref_config2"
GOLDEN = ROOT / "tests" / "golden"
U = 250_000
BLOCK = 1000
KERNELS = {"matmul_skinny_g16x16": "sym", "conv_g16x16": "sym", "fd_stencil_g16x16": "bound", "nbody_g256": "bound"}


def program_keys(kid: str) -> list[int]:
    """schema indices of the GPU program's properties (its .kcp, schema order)"""
    sys.path.insert(0, str(ROOT / "oracle"))
    import kc_oracle as ko
    prog = ko.Program((ROOT / "paper_1604_04997_b200" / "programs" / f"{kid}.kcp").read_text())
    return [k for k, _ in prog.props]


def run(kid, mode, u0, u1, keys):
    with tempfile.NamedTemporaryFile(suffix=".bin") as f:
        r = subprocess.run([str(EXE), kid, mode, str(u0), str(u1), ",".join(map(str, keys)), f.name],
                           capture_output=True, text=True)
        data = Path(f.name).read_bytes()
    return r.returncode, r.stderr, data


def bound_limit(kid, keys):
    """largest u whose bound-mode extraction stays under the reference's cap"""
    lo, hi = 1, 2
    while run(kid, "bound", hi, hi + 1, keys)[0] == 0:
        lo, hi = hi, hi * 2
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if run(kid, "bound", mid, mid + 1, keys)[0] == 0:
            lo = mid
        else:
            hi = mid
    return lo


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=8)
    args = ap.parse_args()
    out = {"note": "sha256 per block of 1000 config-2 points: per point, the GPU program's keys as little-endian "
                   "int128 counts then the fp64 prediction bits, from the reference (oracle/_ref/kcref_config2; "
                   "tests/gen/gen_config2.py)", "block": BLOCK, "kernels": {}}
    for kid, mode in KERNELS.items():
        t0 = time.time()
        keys = program_keys(kid)
        u_end = U + 1 if mode == "sym" else bound_limit(kid, keys) + 1
        cuts = np.linspace(1, u_end, args.procs * 4 + 1).astype(int)
        if mode == "bound":  # cost grows ~u^2: balance the ranges by sqrt spacing
            cuts = np.unique((1 + (u_end - 1) * np.sqrt(np.linspace(0, 1, args.procs * 4 + 1))).astype(int))
        parts = {}
        with cf.ThreadPoolExecutor(args.procs) as ex:
            futs = {ex.submit(run, kid, mode, int(a), int(b), keys): (int(a), int(b))
                    for a, b in zip(cuts[:-1], cuts[1:]) if b > a}
            for f in cf.as_completed(futs):
                rc, err, data = f.result()
                if rc != 0:
                    raise SystemExit(f"{kid} {futs[f]}: rc {rc} {err}")
                parts[futs[f][0]] = data
        blob = b"".join(parts[a] for a in sorted(parts))
        rec = 16 * len(keys) + 8
        n = len(blob) // rec
        assert n == u_end - 1, (kid, n, u_end)
        hashes = [hashlib.sha256(blob[i * rec:min(n, i + BLOCK) * rec]).hexdigest() for i in range(0, n, BLOCK)]
        first = np.frombuffer(blob[:rec], dtype=np.int64)
        out["kernels"][kid] = {"mode": mode, "u_first": 1, "u_last": u_end - 1, "points": n, "keys": keys,
                               "hashes": hashes, "first_record": [int(x) for x in first]}
        print(f"{kid}: {mode}, u = 1..{u_end - 1} ({n} points), {time.time() - t0:.1f} s", flush=True)
    (GOLDEN / "config2_hashes.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
