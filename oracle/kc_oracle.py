"""ORACLE TEST INFRASTRUCTURE -- CPU restatement of the reference hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, and only as the checker. It restates, in exact Python
arithmetic (int / fractions.Fraction, IEEE doubles without FMA):

  CountExpr::evaluate / evaluate_rat / atom_eval   countexpr.cpp:340-383
  CountExpr::str() syntax (prefix)                 countexpr.cpp:385-416
  LinExpr::evaluate / LinCmp::evaluate             linexpr.cpp:83-144
  AssumeCtx::admits                                decide.cpp:153-170
  evaluate_properties                              props.cpp:259-271
  predict                                          model.cpp:95-117
  noiseless_time                                   simdevice.cpp:76-90
  build_design_matrix                              model.cpp:11-35
  fit_weights (min-norm LS on equilibrated cols)   model.cpp:37-93
  geometric_mean_error                             model.cpp:119-133
  keyed_gaussian / splitmix64 / fnv1a              simdevice.cpp:13-46

Parity pinning: tests/test_oracle.py checks this module against the golden
vectors exported by the reference itself (oracle/_ref/kcref_export, built in
place from /root/reference against oracle/shim) -- every count bit-exact and
every prediction bitwise.
"""
from __future__ import annotations

import math
import re
from fractions import Fraction

SCHEMA_CLASSES = ["uniform", "1/1", "1/2", "2/2", "1/3", "2/3", "3/3", "1/4",
                  "2/4", "3/4", "4/4", "1/>4", "2/>4", "3/>4", "4/>4"]


def schema_keys() -> list[str]:
    """schema.cpp:16-38"""
    keys = []
    for d in ("load", "store"):
        for sz in ("s32", "s64", "s128"):
            for c in SCHEMA_CLASSES:
                keys.append(f"mem.global.{d}.{sz}.{c}")
    for sz in ("s32", "s64", "s128"):
        for c in SCHEMA_CLASSES:
            keys.append(f"mem.minls.{sz}.{c}")
    keys.append("mem.local.load")
    for dt in ("f32", "f64"):
        for k in ("addsub", "mul", "div", "pow", "special"):
            keys.append(f"flop.{dt}.{k}")
    keys += ["sync.barrier", "launch.groups", "launch.const"]
    return keys


SCHEMA = schema_keys()
SCHEMA_INDEX = {k: i for i, k in enumerate(SCHEMA)}


class AssumptionViolated(Exception):
    """Errc::assumption_violated (props.cpp:264-266)"""


class NonIntegral(Exception):
    """countexpr.cpp:380-381 logic_error"""


def floor_div(a: int, b: int) -> int:
    """numeric.hpp:24-28 (Python // is already floor division)"""
    return a // b


# ---------------------------------------------------------------------------
# CountExpr prefix text -> evaluator

def _tokens(text: str):
    return re.findall(r"\(|\)|[^\s()]+", text)


def _parse(toks, i):
    if toks[i] == "(":
        i += 1
        out = []
        while toks[i] != ")":
            node, i = _parse(toks, i)
            out.append(node)
        return out, i + 1
    return toks[i], i + 1


def _num(tok: str):
    if re.fullmatch(r"-?\d+(/\d+)?", tok):
        return Fraction(tok)
    return None


def _eval(node, b) -> Fraction:
    if isinstance(node, str):
        c = _num(node)
        if c is not None:
            return c
        if node not in b:
            raise KeyError(f"unbound variable: {node}")
        return Fraction(b[node])
    head, args = node[0], node[1:]
    if head == "+":
        return sum((_eval(a, b) for a in args), Fraction(0))
    if head == "*":
        r = Fraction(1)
        for a in args:
            r *= _eval(a, b)
        return r
    if head == "^":
        v = _eval(args[0], b)
        r = Fraction(1)
        for _ in range(int(args[1])):       # repeated multiply, countexpr.cpp:371
            r *= v
        return r
    if head == "floordiv":                   # countexpr.cpp:348-349
        q = _eval(args[0], b) / Fraction(int(args[1]))
        return Fraction(floor_div(q.numerator, q.denominator))
    if head in ("min", "max"):               # countexpr.cpp:350-358
        best = _eval(args[0], b)
        for a in args[1:]:
            v = _eval(a, b)
            if (v < best) if head == "min" else (v > best):
                best = v
        return best
    raise ValueError(f"unknown operator {head}")


class CountExpr:
    def __init__(self, text: str):
        self.text = text
        toks = _tokens(text)
        self.node, n = _parse(toks, 0)
        if n != len(toks):
            raise ValueError(f"trailing tokens in {text!r}")

    def evaluate_rat(self, b) -> Fraction:
        return _eval(self.node, b)

    def evaluate(self, b) -> int:
        v = self.evaluate_rat(b)
        if v.denominator != 1:
            raise NonIntegral(f"count evaluated to non-integer {v}")
        return v.numerator


# ---------------------------------------------------------------------------
# LinCmp text (linexpr.cpp:97-155) -> evaluator

_LIN_TOK = re.compile(r"\s*(//|\d+|[A-Za-z_]\w*|[-+*/()%<>=]=?|==)")


class LinCmp:
    def __init__(self, text: str):
        self.text = text
        if " % " in text:
            lhs, rest = text.split(" % ", 1)
            mod, rem = rest.split(" == ")
            self.div = True
            self.lhs, self.rhs = lhs, "0"
            self.mod, self.rem, self.op = int(mod), int(rem), None
        else:
            for op in (" <= ", " >= ", " == ", " < ", " > "):
                if op in text:
                    lhs, rhs = text.split(op, 1)
                    break
            else:
                raise ValueError(f"no comparison in {text!r}")
            self.div, self.op = False, op.strip()
            self.lhs, self.rhs = lhs, rhs

    @staticmethod
    def _lin(text: str, env) -> Fraction:
        # LinExpr::evaluate (linexpr.cpp:83-97): affine terms, rational
        # coefficients "a/b*v", floordiv terms "(inner)//den"
        toks = [t for t in _LIN_TOK.findall(text) if t]
        pos = 0

        def peek():
            return toks[pos] if pos < len(toks) else None

        def take():
            nonlocal pos
            pos += 1
            return toks[pos - 1]

        def factor():
            if peek() == "(":
                take()
                inner = expr()
                assert take() == ")"
                assert take() == "//"
                den = int(take())
                return Fraction(floor_div(inner.numerator, inner.denominator * den))
            name = take()
            return Fraction(env[name])

        def term():
            if peek() is not None and peek().isdigit():
                c = Fraction(int(take()))
                if peek() == "/":
                    take()
                    c /= int(take())
                if peek() == "*":
                    take()
                    return c * factor()
                return c
            return factor()

        def expr():
            sign = 1
            if peek() == "-":
                take()
                sign = -1
            acc = sign * term()
            while peek() in ("+", "-"):
                s = 1 if take() == "+" else -1
                acc += s * term()
            return acc

        v = expr()
        return v

    def evaluate(self, env) -> bool:
        """linexpr.cpp:128-144"""
        if self.div:
            v = self._lin(self.lhs, env)
            if v.denominator != 1:
                raise NonIntegral(f"expected integral rational, got {v}")
            iv = v.numerator
            return ((iv % self.mod) + self.mod) % self.mod == self.rem
        l, r = self._lin(self.lhs, env), self._lin(self.rhs, env)
        return {"<": l < r, "<=": l <= r, ">": l > r, ">=": l >= r, "==": l == r}[self.op]


# ---------------------------------------------------------------------------
# programs (kernelcost-program v1 text)

class Program:
    def __init__(self, text: str):
        self.params: list[str] = []
        self.assume: list[LinCmp] = []
        self.props: list[tuple[int, CountExpr]] = []
        self.name = ""
        for line in text.splitlines():
            line = line.strip()
            if not line or line == "kernelcost-program v1" or line == "end":
                continue
            kw, _, rest = line.partition(" ")
            if kw == "kernel":
                self.name = rest
            elif kw == "param":
                self.params.append(rest)
            elif kw == "assume":
                self.assume.append(LinCmp(rest))
            elif kw == "prop":
                key, _, expr = rest.partition(" ")
                self.props.append((SCHEMA_INDEX[key], CountExpr(expr)))
        self.props.sort(key=lambda kv: kv[0])

    def admits(self, b) -> bool:
        """AssumeCtx::admits (decide.cpp:153-170): every recorded constraint
        (the distilled per-parameter facts are implied by the raw ones),
        then parameters >= 0."""
        for c in self.assume:
            if not c.evaluate(b):
                return False
        return all(b[p] >= 0 for p in self.params)

    def evaluate_properties(self, b) -> dict[int, int]:
        """props.cpp:259-271 -> {schema index: exact count} (nonzero keys)"""
        for p in self.params:
            if p not in b:
                raise KeyError(f"binding missing parameter '{p}'")
        if not self.admits(b):
            raise AssumptionViolated("binding violates the kernel's assumptions")
        return {k: e.evaluate(b) for k, e in self.props}


def predict(alpha149, counts: dict[int, int]) -> float:
    """model.cpp:95-117: schema order, skip zero counts, part = a*count;
    seconds += part (no FMA: Python floats round each operation)."""
    s = 0.0
    for j in sorted(counts):
        c = counts[j]
        if c == 0:
            continue
        part = alpha149[j] * float(c)      # float(int) rounds to nearest even
        s += part
    return s


def noiseless_time(alpha149, counts: dict[int, int]) -> float:
    """simdevice.cpp:76-90: schema order, skip zero weights"""
    t = 0.0
    for j in range(len(alpha149)):
        if alpha149[j] == 0.0:
            continue
        t += alpha149[j] * float(counts.get(j, 0))
    return t


def build_design_matrix(cases):
    """model.cpp:11-35: rows p_j / T, covered = any nonzero."""
    import numpy as np
    if not cases:
        raise ValueError("E_EMPTY: no fit cases")
    X = np.zeros((len(cases), len(SCHEMA)))
    for r, (counts, t) in enumerate(cases):
        if not t > 0.0:
            raise ValueError("E_NONPOSITIVE_TIME")
        for j, c in counts.items():
            if c != 0:
                X[r, j] = float(c) / t
    covered = (X != 0).any(axis=0)
    return X, covered


def fit_weights(X, covered):
    """model.cpp:37-93 with numpy's SVD least squares standing in for Eigen's
    COD (both give the minimum-norm solution): equilibrate covered columns by
    1/max|col|, solve, alpha = x * scale, residuals 1 - A x."""
    import numpy as np
    cols = np.flatnonzero(covered)
    alpha = np.zeros(X.shape[1])
    resid = np.ones(X.shape[0])
    if len(cols):
        A = X[:, cols].copy()
        m = np.abs(A).max(axis=0)
        scale = np.where(m > 0, 1.0 / m, 1.0)
        A *= scale
        x, *_ = np.linalg.lstsq(A, np.ones(X.shape[0]), rcond=None)
        resid = 1.0 - A @ x
        alpha[cols] = x * scale
    return alpha, float(resid @ resid), resid


def geometric_mean_error(pairs) -> float:
    """model.cpp:119-133"""
    if not pairs:
        raise ValueError("E_EMPTY")
    s = 0.0
    for pred, actual in pairs:
        if not actual > 0.0:
            raise ValueError("E_NONPOSITIVE_TIME")
        rel = abs(pred - actual) / actual
        s += math.log(max(rel, 1e-12))
    return math.exp(s / len(pairs))


M64 = (1 << 64) - 1


def splitmix64(state: int) -> tuple[int, int]:
    """simdevice.cpp:15-21 -> (new state, output)"""
    state = (state + 0x9E3779B97F4A7C15) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def fnv1a(s: str) -> int:
    """simdevice.cpp:23-30"""
    h = 1469598103934665603
    for c in s.encode():
        h ^= c
        h = (h * 1099511628211) & M64
    return h


def keyed_gaussian(seed: int, key: str, counter: int) -> float:
    """simdevice.cpp:37-46"""
    st = fnv1a(key) ^ ((seed * 0x9E3779B97F4A7C15) & M64) ^ ((counter * 0xD1342543DE82EF95) & M64)
    st, a = splitmix64(st)
    st, b = splitmix64(st)
    u1 = (a >> 11) * 2.0 ** -53
    u2 = (b >> 11) * 2.0 ** -53
    if u1 <= 0.0:
        u1 = 2.0 ** -53
    return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * 3.14159265358979323846 * u2)


def simdev_reference_alpha() -> list[float]:
    """SimDevice::reference() (simdevice.cpp:48-74): Table 2 weights"""
    a = [0.0] * len(SCHEMA)
    for k, v in {
        "flop.f32.addsub": 6.81e-13, "flop.f32.mul": 5.68e-13, "flop.f32.pow": 3.91e-13,
        "flop.f32.special": 1.61e-12, "mem.local.load": -1.76e-12,
        "mem.global.load.s32.1/1": 8.27e-12, "mem.global.load.s32.2/2": 9.82e-13,
        "mem.global.load.s32.2/3": 2.89e-11, "mem.global.load.s32.3/3": 9.30e-13,
        "mem.global.load.s32.4/>4": 2.67e-12, "mem.global.store.s32.1/1": 6.52e-12,
        "mem.global.store.s32.4/>4": 3.55e-10, "mem.minls.s32.1/1": -6.63e-12,
        "sync.barrier": 4.26e-11, "launch.groups": 3.75e-09, "launch.const": 1.29e-04,
    }.items():
        a[SCHEMA_INDEX[k]] = v
    return a


def parse_binding(s: str) -> dict:
    """csvio.cpp:86-102"""
    b = {}
    if not s:
        return b
    for part in s.split(";"):
        k, _, v = part.partition("=")
        b[k] = int(v)
    return b


def read_any_csv(path, discard: int = 4):
    """kernelcost.cpp:116-126: measurement CSV, or raw runs reduced like
    reduce_raw_runs (csvio.cpp:192-225). Returns [(kernel, binding, time)]."""
    lines = [ln.rstrip("\r") for ln in open(path).read().splitlines() if ln.strip()]
    header, rows = lines[0], [ln.split(",") for ln in lines[1:]]
    if header == "kernel,binding,group_config,time_s":
        return [(r[0], parse_binding(r[1]), float(r[3])) for r in rows]
    assert header == "kernel,binding,group_config,run_index,time_s", header
    groups = {}
    for r in rows:
        b = parse_binding(r[1])
        key = (r[0], ";".join(f"{k}={v}" for k, v in sorted(b.items())), r[2])
        groups.setdefault(key, []).append((int(r[3]), float(r[4])))
    out = []
    for key in sorted(groups):
        times = [t for _, t in sorted(groups[key])]
        if len(times) <= discard:
            raise ValueError("E_INVALID_ARGUMENT: not enough runs")
        out.append((key[0], parse_binding(key[1]), min(times[discard:])))
    return out
