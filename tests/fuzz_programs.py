"""Seeded generator of random kernelcost-program texts: polynomials with
rational coefficients over floordiv / min / max atoms and congruence /
relational / floordiv assumptions -- the whole CountExpr / LinCmp surface
(countexpr.hpp:20-117, linexpr.hpp:19-77), not just what the bundled suite
happens to produce. Used by the CPU and GPU fuzz tests."""
import random

PARAMS = ["n", "m", "k"]
KEYS = ["mem.global.load.s32.1/1", "mem.global.store.s32.1/1", "mem.local.load", "flop.f32.addsub",
        "flop.f64.mul", "sync.barrier", "launch.groups", "launch.const", "mem.minls.s64.2/3"]


def _coef(rng, allow_frac=True):
    num = rng.choice([1, 1, 1, 2, 3, 5, 7, 9, 16, 48, -1, -3])
    if allow_frac and rng.random() < 0.35:
        return f"{num}/{rng.choice([2, 3, 4, 6, 8, 12])}"
    return str(num)


def _affine(rng, params):
    terms = [f"(* {_coef(rng, False)} {p})" for p in rng.sample(params, rng.randint(1, len(params)))]
    if rng.random() < 0.5:
        terms.append(str(rng.randint(-5, 9)))
    return terms[0] if len(terms) == 1 else "(+ " + " ".join(terms) + ")"


def _atom(rng, params, depth):
    r = rng.random()
    if r < 0.55 or depth > 1:
        return rng.choice(params)
    if r < 0.8:
        inner = _affine(rng, params) if rng.random() < 0.7 else _poly(rng, params, depth + 1)
        return f"(floordiv {inner} {rng.choice([2, 3, 4, 5, 7, 16])})"
    args = " ".join(_affine(rng, params) for _ in range(rng.randint(2, 3)))
    return f"({rng.choice(['min', 'max'])} {args})"


def _mono(rng, params, depth):
    fs = []
    for _ in range(rng.randint(1, 3)):
        a = _atom(rng, params, depth)
        if rng.random() < 0.2:
            a = f"(^ {a} 2)"
        fs.append(a)
    return "(* " + _coef(rng) + " " + " ".join(fs) + ")"


def _poly(rng, params, depth=0):
    terms = [_mono(rng, params, depth) for _ in range(rng.randint(1, 3))]
    if rng.random() < 0.4:
        terms.append(_coef(rng))
    return terms[0] if len(terms) == 1 else "(+ " + " ".join(terms) + ")"


def random_program(seed: int) -> str:
    rng = random.Random(seed)
    params = PARAMS[: rng.randint(1, 3)]
    lines = ["kernelcost-program v1", f"kernel fuzz_{seed}"] + [f"param {p}" for p in params]
    for p in params:
        r = rng.random()
        if r < 0.4:
            lines.append(f"assume {p} % {rng.choice([2, 4, 6, 8, 12, 16])} == 0")
        elif r < 0.55:
            mod = rng.choice([3, 5, 6])
            lines.append(f"assume {p} % {mod} == {rng.randint(0, mod - 1)}")
        if rng.random() < 0.5:
            lines.append(f"assume {p} >= {rng.randint(0, 20)}")
    if len(params) > 1 and rng.random() < 0.4:
        lines.append(f"assume {params[0]} + 2*{params[1]} >= 7")
    if rng.random() < 0.2:
        lines.append(f"assume 1/2*{params[0]} <= 1000000000000")
    if rng.random() < 0.2:
        lines.append(f"assume ({params[0]} + 1)//3 >= 1")
    for key in sorted(rng.sample(KEYS, rng.randint(2, 6)), key=KEYS.index):
        lines.append(f"prop {key} {_poly(rng, params)}")
    lines.append("end")
    # schema order of prop lines is not required by either parser
    return "\n".join(lines) + "\n"


def random_bindings(seed: int, params, count: int):
    rng = random.Random(seed * 7919 + 1)
    out = []
    for i in range(count):
        r = rng.random()
        b = {}
        for p in params:
            if r < 0.5:
                v = rng.randint(0, 60)
            elif r < 0.8:
                v = rng.randint(0, 2_000_000)
            elif r < 0.95:
                v = rng.randint(0, 1 << rng.choice([33, 40, 48, 62]))
            else:
                v = -rng.randint(0, 50)
            b[p] = v
        # bias toward congruence-satisfying values so many points are admissible
        if rng.random() < 0.6:
            b = {p: v - v % 48 if v >= 48 else v for p, v in b.items()}
        out.append(b)
    return out
