"""Random kernels (the reference's kernel IR text) for the enumeration
oracle's parity fuzz: loop nests with parametric / triangular bounds,
guards (relational and divisibility), 1-3D global arrays in both layouts
with strided / offset / transposed indices, local arrays, barriers.
  python tests/gen/gen_enum_kernels.py > tests/golden/enum_random_kernels.txt
Then `oracle/_ref/kcref_export --enum-kernels <that file> tests/golden/enum_random.json`
records the reference's enumerate_points for each kernel at small bindings."""
import random


def kernel(seed):
    r = random.Random(seed)
    two = r.random() < 0.6
    params = ["n", "m"] if two else ["n"]
    assume = ["n >= 1"] + (["m >= 1"] if two else [])
    if r.random() < 0.3:
        assume.append("n % 2 == 0")
    L = [f"kernel x_r{seed}", "param " + ", ".join(params), "assume " + " and ".join(assume)]
    ndim = r.choice([1, 1, 2, 2, 3])
    lay = r.choice(["row_major", "column_major"])
    pe = lambda: r.choice(params)  # noqa: E731
    shape = ", ".join(f"{pe()} + {r.randint(2, 9)}" for _ in range(ndim))
    dt = r.choice(["f32", "f64"])
    L.append(f"array a : {dt} [{shape}] global {lay} in")
    L.append(f"array o : {dt} [{pe()} + 8, 8] global {r.choice(['row_major', 'column_major'])} out")
    use_t = r.random() < 0.4
    if use_t:
        L.append(f"array t : {dt} [16] local row_major temp")
    grp = r.choice(["1", "n // 2", f"{pe()} // 3", "2"])
    L.append(f"axis g0 = group(0) extent {grp}")
    lx = r.choice([1, 2, 3, 4])
    L.append(f"axis l0 = local(0) extent {lx}")
    vars_ = ["g0", "l0"]
    body = []
    depth = 0
    if use_t:
        body.append("t[l0] = a[" + ", ".join(["l0"] + ["0"] * (ndim - 1)) + "]")
        body.append("barrier")
    nloops = r.choice([1, 1, 2, 2, 3])
    for k in range(nloops):
        v = "ijk"[k]
        lo = "0" if k == 0 or r.random() < 0.5 else r.choice(vars_[2:] or ["0"])
        hi = r.choice([pe(), f"{pe()} + 1"] + ([f"{vars_[-1]} + 1", f"{vars_[-1]} + 2"] if k else []))
        body.append(f"loop {v} = {lo} .. {hi}")
        vars_.append(v)
        depth += 1
        if r.random() < 0.35:
            g = r.choice([f"{v} < {pe()}", f"{v} >= 1", f"{v} % {r.randint(2, 3)} == {r.randint(0, 1)}",
                          f"2*{v} <= {pe()} + 1", f"l0 == {r.randint(0, lx - 1)}"])
            body.append(f"guard {g}")
            depth += 1

    def idx(dim_count):
        out = []
        for _ in range(dim_count):
            terms = [f"{r.randint(1, 3)}*{x}" if r.random() < 0.3 else x
                     for x in r.sample(vars_, k=r.randint(1, min(2, len(vars_))))]
            terms.append(str(r.randint(0, 2)))
            out.append(" + ".join(terms))
        return ", ".join(out)
    rhs = f"a[{idx(ndim)}] * 2.0"
    if r.random() < 0.5:
        rhs += f" + a[{idx(ndim)}]"
    if use_t:
        rhs += " + t[l0]"
    body.append(f"o[{idx(2)}] = {rhs}")
    body += ["end"] * depth
    return "\n".join(L + body) + "\n"


if __name__ == "__main__":
    print("\n----\n".join(kernel(s) for s in range(120)))
