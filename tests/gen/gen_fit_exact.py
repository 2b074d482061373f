"""Exact minimum-norm least-squares solutions of the reference's fit
fixtures -> tests/golden/fit_exact.json (test infrastructure).

fit_weights (model.cpp:37-93) solves min || 1 - X alpha || in the minimum-
norm sense over the covered columns of the double-precision design
X_ij = double(count_ij) / T_i (model.cpp:29). Every X_ij is a dyadic
rational, so the solution of that exact problem is computable exactly:
X = M / 2^S with integer M, G = M^T M and b = 2^S M^T 1 in integers, then
x = x_p - N (N^T N)^-1 N^T x_p with x_p a particular solution of G x = b
and N a basis of null(G) = null(X) (the min-norm solution is orthogonal to
it), all in fractions.Fraction. Column equilibration (model.cpp:71-76) does
not change the min-norm solution set's image alpha for full-rank designs;
for rank-deficient ones the reference minimises the norm of the
EQUILIBRATED x, so the null-space projection is done in the scaled
coordinates x_j = alpha_j * max|col_j|, exactly as model.cpp does.

The fixtures: the synthetic fits (fit_synthetic.json), the measurement-suite
design (suite_cases.json, 390 rows) and the two CLI campaign CSVs
(meas_sigma0.csv, raw_runs_sigma002.csv; rows from the oracle's counts).

    python tests/gen/gen_fit_exact.py
"""
from __future__ import annotations

import json
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle"))
import kc_oracle as ko  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"


def hexf(s):
    return float.fromhex(s)


def exact_min_norm_rational(rows: list[list[Fraction]]):
    """The same over an exact rational design (e.g. x_ij = count_ij / T_i
    unrounded): for a design whose columns are exactly dependent (the tiled
    matmul's 9 keys over 3 monomials) the rounded double rows are full rank
    at the 1e-16 level, and only the unrounded design has the min-norm
    solution a rank-revealing solver (the reference's COD) approximates."""
    F = len(rows[0])
    cm = [max(abs(r[j]) for r in rows) for j in range(F)]
    G = [[Fraction(0)] * F for _ in range(F)]
    b = [Fraction(0)] * F
    for r in rows:
        d = [r[j] / cm[j] if cm[j] else Fraction(0) for j in range(F)]
        for j in range(F):
            if d[j] == 0:
                continue
            b[j] += d[j]
            for k in range(j, F):
                G[j][k] += d[j] * d[k]
    for j in range(F):
        for k in range(j):
            G[j][k] = G[k][j]
    x, rank = _min_norm_normal(G, b, F)
    return [x[j] / cm[j] if cm[j] else Fraction(0) for j in range(F)], rank


def exact_min_norm(X: np.ndarray) -> list[Fraction]:
    """min-norm argmin || 1 - D x ||, D = X / colmax (exactly: colmax is a
    double, 1/colmax is applied exactly as a rational), returned as
    alpha = x / colmax."""
    N, F = X.shape
    cm = [Fraction(float(v)) for v in np.abs(X).max(axis=0)]
    # integer image of X: X = M / 2^S
    e_min = int(np.frexp(X[X != 0]).__getitem__(1).min()) if (X != 0).any() else 0
    S = 60 - e_min
    M = [[int(np.ldexp(X[i, j], S)) for j in range(F)] for i in range(N)]
    for i in range(0, N, max(1, N // 50)):
        for j in range(F):
            assert Fraction(M[i][j], 2 ** S) == Fraction(float(X[i, j]))
    Gi = [[0] * F for _ in range(F)]
    bi = [0] * F
    for row in M:
        for j in range(F):
            rj = row[j]
            if rj == 0:
                continue
            bi[j] += rj
            for k in range(j, F):
                Gi[j][k] += rj * row[k]
    for j in range(F):
        for k in range(j):
            Gi[j][k] = Gi[k][j]
    # scaled coordinates: D = X diag(1/cm), x = diag(cm) alpha.
    # (D^T D) x = D^T 1  <=>  diag(1/cm) G diag(1/cm) x = diag(1/cm) b
    G = [[Fraction(Gi[j][k], 2 ** (2 * S)) / (cm[j] * cm[k]) for k in range(F)] for j in range(F)]
    b = [Fraction(bi[j], 2 ** S) / cm[j] for j in range(F)]
    x, rank = _min_norm_normal(G, b, F)
    return [x[j] / cm[j] for j in range(F)], rank


def _min_norm_normal(G, b, F):
    """min-norm solution of the consistent system G x = b (G = D^T D)"""
    # RREF of [G | b]
    A = [G[j][:] + [b[j]] for j in range(F)]
    piv_cols, r = [], 0
    for c in range(F):
        p = next((i for i in range(r, F) if A[i][c] != 0), None)
        if p is None:
            continue
        A[r], A[p] = A[p], A[r]
        pv = A[r][c]
        A[r] = [v / pv for v in A[r]]
        for i in range(F):
            if i != r and A[i][c] != 0:
                f = A[i][c]
                A[i] = [a - f * bb for a, bb in zip(A[i], A[r])]
        piv_cols.append(c)
        r += 1
        if r == F:
            break
    xp = [Fraction(0)] * F
    for i, c in enumerate(piv_cols):
        xp[c] = A[i][F]
    free = [c for c in range(F) if c not in piv_cols]
    # null space basis: one vector per free column
    Nb = []
    for f in free:
        v = [Fraction(0)] * F
        v[f] = Fraction(1)
        for i, c in enumerate(piv_cols):
            v[c] = -A[i][f]
        Nb.append(v)
    x = xp
    if Nb:
        k = len(Nb)
        NtN = [[sum(a * b2 for a, b2 in zip(Nb[i], Nb[j])) for j in range(k)] for i in range(k)]
        Ntx = [sum(a * b2 for a, b2 in zip(Nb[i], xp)) for i in range(k)]
        # solve NtN t = Ntx
        Aug = [NtN[i][:] + [Ntx[i]] for i in range(k)]
        for c in range(k):
            p = next(i for i in range(c, k) if Aug[i][c] != 0)
            Aug[c], Aug[p] = Aug[p], Aug[c]
            pv = Aug[c][c]
            Aug[c] = [v / pv for v in Aug[c]]
            for i in range(k):
                if i != c and Aug[i][c] != 0:
                    f = Aug[i][c]
                    Aug[i] = [a - f * bb for a, bb in zip(Aug[i], Aug[c])]
        t = [Aug[i][k] for i in range(k)]
        x = [xp[j] - sum(t[i] * Nb[i][j] for i in range(k)) for j in range(F)]
    return x, len(piv_cols)


def suite_design():
    cases = [c for c in json.loads((GOLDEN / "suite_cases.json").read_text())["cases"] if c["role"] == "measurement"]
    rows = [({ko.SCHEMA_INDEX[k]: int(v) for k, v in c["counts"].items()}, hexf(c["time_s"][1])) for c in cases]
    X, cov = ko.build_design_matrix(rows)
    cols = np.flatnonzero(cov)
    return [ko.SCHEMA[c] for c in cols], np.ascontiguousarray(X[:, cols])


def csv_design(name):
    recs = ko.read_any_csv(GOLDEN / name)
    progs = {}
    rows = []
    for kernel, binding, t in recs:
        if kernel not in progs:
            progs[kernel] = ko.Program((ROOT / "paper_1604_04997_b200" / "programs" / f"{kernel}.kcp").read_text())
        rows.append((progs[kernel].evaluate_properties(binding), t))
    X, cov = ko.build_design_matrix(rows)
    cols = np.flatnonzero(cov)
    return [ko.SCHEMA[c] for c in cols], np.ascontiguousarray(X[:, cols])


def main():
    out = {"note": "exact min-norm least-squares solutions of the double-precision designs "
                   "(tests/gen/gen_fit_exact.py); alpha as hex doubles (correctly rounded)", "fits": []}
    designs = []
    for fit in json.loads((GOLDEN / "fit_synthetic.json").read_text())["fits"]:
        counts = np.array(fit["counts"], dtype=np.float64)
        times = np.array([hexf(t) for t in fit["times"]])
        designs.append((fit["name"], fit["keys"], counts / times[:, None], [hexf(a) for a in fit["alpha"]]))
    keys, X = suite_design()
    fs = json.loads((GOLDEN / "fit_suite.json").read_text())
    designs.append(("suite_measurement_390", keys, X, [hexf(fs["alpha"][k][1]) if k in fs["alpha"] else 0.0
                                                        for k in keys]))
    cli = json.loads((GOLDEN / "cli_fit_eval.json").read_text())
    for name in ("meas_sigma0.csv", "raw_runs_sigma002.csv"):
        keys, X = csv_design(name)
        designs.append((f"cli_{name}", keys, X, [hexf(cli[name]["alpha"][k]) if k in cli[name]["alpha"] else 0.0
                                                 for k in keys]))
    for name, keys, X, ref in designs:
        alpha, rank = exact_min_norm(X)
        a = [float(v) for v in alpha]
        rel = [abs(r - e) / abs(e) if e != 0 else abs(r) for r, e in zip(ref, a)]
        out["fits"].append({"name": name, "keys": keys, "rank": rank, "rows": int(X.shape[0]),
                            "alpha_exact": [v.hex() for v in a],
                            "reference_cod_rel_diff": rel})
        print(f"{name}: rows {X.shape[0]} cols {X.shape[1]} rank {rank}  max |ref COD - exact| / |exact| = "
              f"{max(r for r, e in zip(rel, a) if e != 0):.2e}")
    (GOLDEN / "fit_exact.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
