"""Random kernels whose statement domains use floor division over DOMAIN
variables in loop bounds -- `j = i // 3 .. (i + 1) // 2 + 1`,
`(i + n) // 3 + 1` -- (the reference's parser allows `//` only in extents
and loop bounds) -- the shapes the reference's enumerator walks with its
generic Walker (enumerate.cpp:31-90) instead of the compiled rows. For the
GPU enumeration oracle's parity fuzz.
  python tests/gen/gen_enum_fd_kernels.py > tests/golden/enum_fd_kernels.txt
  oracle/_ref/kcref_export --enum-kernels tests/golden/enum_fd_kernels.txt tests/golden/enum_fd.json"""
import random


def kernel(seed):
    r = random.Random(1000 + seed)
    two = r.random() < 0.5
    params = ["n", "m"] if two else ["n"]
    assume = ["n >= 1"] + (["m >= 1"] if two else [])
    L = [f"kernel x_fd{seed}", "param " + ", ".join(params), "assume " + " and ".join(assume)]
    pe = lambda: r.choice(params)  # noqa: E731
    ndim = r.choice([1, 2])
    lay = r.choice(["row_major", "column_major"])
    shape = ", ".join(f"{pe()} + {r.randint(4, 9)}" for _ in range(ndim))
    L.append(f"array a : f32 [{shape}] global {lay} in")
    L.append(f"array o : f32 [{pe()} + 8, 8] global row_major out")
    L.append(f"axis g0 = group(0) extent {r.choice(['1', '2', 'n // 2'])}")
    lx = r.choice([1, 2, 4])
    L.append(f"axis l0 = local(0) extent {lx}")
    body, depth, vars_ = [], 0, ["g0", "l0"]
    nloops = r.choice([2, 2, 3])
    for k in range(nloops):
        v = "ijk"[k]
        if k == 0:
            hi = r.choice([pe(), f"{pe()} + 1"])
            lo = "0"
        else:
            p = vars_[-1]
            hi = r.choice([f"({p} + 1) // 2 + 1", f"{p} // 2 + 1", f"({p} + {pe()}) // 3 + 1", f"{p} + 1"])
            lo = r.choice(["0", "0", f"{p} // 3"])
        body.append(f"loop {v} = {lo} .. {hi}")
        vars_.append(v)
        depth += 1
        # no guards: the reference's FastDomain returns from its guard loop
        # once a floordiv-over-domain bound failed to compile, keeping
        # ok = true with incomplete rows (enumerate.cpp:204-214) -- 0 points;
        # guarded statements are checked against a brute force instead
        # (tests/test_enumerate.py::test_enumerate_floordiv_with_guards_brute_force)

    def idx(dims):
        out = []
        for _ in range(dims):
            x = r.choice(vars_[2:])
            y = r.choice(vars_)
            out.append(r.choice([f"2*{x} + {y}", f"{x} + {y}", f"{x}", f"{y} + 1", f"3*{x} + 1"]))
        return ", ".join(out)
    rhs = f"a[{idx(ndim)}] * 2.0"
    if r.random() < 0.5:
        rhs += f" + a[{idx(ndim)}]"
    body.append(f"o[{idx(2)}] = {rhs}")
    body += ["end"] * depth
    return "\n".join(L + body) + "\n"


if __name__ == "__main__":
    print("\n----\n".join(kernel(s) for s in range(60)))
