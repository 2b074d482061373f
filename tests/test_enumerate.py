"""GPU enumeration oracle (kcg_enumerate_points) against the reference's own
enumerate_points (enumerate.cpp:371-456): the golden tallies exported by
oracle/kcref_export (3 oracle-lattice draws of every suite kernel plus
triangular / guarded / divisibility-guarded / strided test kernels, counts
and visited points), and -- at sizes the CPU enumerator cannot reach --
against the symbolic programs evaluated on the GPU (the symbolic counts of
the reference front end, and the derived fd_stencil / nbody closed forms of
SURVEY §8f row 1)."""
import pytest

from conftest import PROGRAMS, load_golden

import paper_1604_04997_b200 as kc  # noqa: E402
from paper_1604_04997_b200 import _capi  # noqa: E402

ENUM = PROGRAMS / "enum"


def test_every_enum_program_parses():
    files = sorted(ENUM.glob("*.kce"))
    assert len(files) >= 61 + 4
    for f in files:
        p = kc.EnumProgram.from_file(f)
        assert p.params, f.name


def test_enum_text_errors_are_parse_errors():
    with pytest.raises(kc.KcgError) as e:
        kc.EnumProgram("kernelcost-enum v1\nkernel k\nparam n\nstmt assign\nvar i 0 | n\nbogus\nendstmt\nend\n")
    assert e.value.code == _capi.E_PARSE
    with pytest.raises(kc.KcgError):
        kc.EnumProgram("kernelcost-program v1\nend\n")
    with pytest.raises(kc.KcgError):  # access to an undeclared array
        kc.EnumProgram("kernelcost-enum v1\nkernel k\nparam n\nstmt assign\nvar i 0 | n\n"
                       "access a load 1 | i\nendstmt\nend\n")


def test_enumerate_without_device_fails_loudly():
    import ctypes
    p = kc.load_enum_program("vecop_s1_g256")
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("device present")
    except ImportError:
        pass
    n = kc.schema_size()
    lo, hi = (ctypes.c_int64 * n)(), (ctypes.c_int64 * n)()
    b = (ctypes.c_int64 * 1)(256)
    rc = _capi.lib().kcg_enumerate_points(p._h, b, 0, lo, hi, None, None)
    assert rc == _capi.E_CUDA


def _cases():
    return load_golden("enum_points.json")["cases"]


@pytest.mark.gpu
def test_enumerate_matches_reference_goldens():
    progs = {}
    n_ok = 0
    for c in _cases():
        k = c["kernel"]
        if k not in progs:
            progs[k] = kc.load_enum_program(k)
        b = {p: int(v) for p, v in c["binding"].items()}
        if c["status"] != "ok":
            with pytest.raises(kc.KcgError) as e:
                progs[k].enumerate_points(b)
            assert e.value.name == c["status"], (k, b)
            continue
        counts, points = progs[k].enumerate_points(b)
        want = {key: int(v) for key, v in c["counts"].items()}
        assert counts == want, (k, b)
        assert points == int(c["points"]), (k, b)
        n_ok += 1
    assert n_ok >= 250


@pytest.mark.gpu
def test_enumerate_cap_exceeded():
    p = kc.load_enum_program("fd_stencil_g16x16")
    _, pts = p.enumerate_points({"n": 64})
    with pytest.raises(kc.KcgError) as e:
        p.enumerate_points({"n": 64}, cap=pts - 1)
    assert e.value.code == _capi.E_CAP_EXCEEDED
    assert p.enumerate_points({"n": 64}, cap=pts)[1] == pts


def _symbolic_counts(kid, b):
    import torch
    prog = kc.load_program(kid)
    cols = {p: torch.tensor([b[p]], dtype=torch.int64, device="cuda") for p in prog.params}
    bb = kc.evaluate_properties(prog, cols, wide=True)
    torch.cuda.synchronize()
    assert int(bb.status[0]) == 0
    keys = kc.schema_keys()
    return {keys[k]: bb.counts_int(j, 0) for j, k in enumerate(prog.props) if bb.counts_int(j, 0)}


@pytest.mark.gpu
@pytest.mark.parametrize("kid,b", [
    ("fd_stencil_g16x16", {"n": 4096}),      # 1.2e8 visited points; CPU cap is 2e7
    ("nbody_g256", {"n": 8192}),             # 6.9e7
    ("matmul_tiled_g16x16", {"n": 512, "m": 256, "l": 768}),
    ("conv_g16x16", {"n": 256}),
    ("transpose_tile_g16x16", {"n": 4096}),
    ("vecop_s3_g192", {"n": 192 * 100000}),
])
def test_enumerate_equals_symbolic_beyond_cpu_cap(kid, b):
    """Brute force on the GPU == the closed forms (derived for fd_stencil /
    nbody, the front end's symbolic PV otherwise), bit-exact, far past the
    reference's 2e7-point enumeration cap."""
    counts, points = kc.load_enum_program(kid).enumerate_points(b)
    assert points > 0
    assert counts == _symbolic_counts(kid, b)


def _random_kernels():
    return [k for k in load_golden("enum_random.json")["kernels"] if "cases" in k]


def test_random_kernel_enum_texts_parse():
    ks = _random_kernels()
    assert len(ks) == 120
    for k in ks:
        kc.EnumProgram(k["enum_text"])


@pytest.mark.gpu
def test_enumerate_random_kernels_match_reference():
    """120 random kernels (tests/gen/gen_enum_kernels.py: parametric and
    triangular loop nests, relational / divisibility / lane guards, 1-3D
    arrays in both layouts, strided and offset indices, local arrays,
    barriers) x up to 24 bindings: counts, visited points and errors equal
    the reference's enumerate_points (tests/golden/enum_random.json)."""
    n_ok = 0
    for k in _random_kernels():
        p = kc.EnumProgram(k["enum_text"])
        for c in k["cases"]:
            b = {q: int(v) for q, v in c["binding"].items()}
            if c["status"] != "ok":
                with pytest.raises(kc.KcgError) as e:
                    p.enumerate_points(b)
                assert e.value.name == c["status"], (k["id"], b)
                continue
            counts, points = p.enumerate_points(b)
            want = {key: int(v) for key, v in c["counts"].items()}
            assert counts == want, (k["id"], b, counts, want)
            assert points == int(c["points"]), (k["id"], b, points, c["points"])
            n_ok += 1
    assert n_ok > 1500


def _scaled_cases():
    """Every suite kernel at its largest golden binding scaled by an integer
    k (divisibility is preserved) so that the walk visits ~1e7-3e8 points:
    far past the reference's 2e7 cap for most kernels."""
    best = {}
    for c in _cases():
        if c["status"] == "ok" and (c["kernel"] not in best or int(c["points"]) > int(best[c["kernel"]]["points"])):
            best[c["kernel"]] = c
    out = []
    for kid, c in sorted(best.items()):
        if not (PROGRAMS / f"{kid}.kcp").exists():  # x_* test kernels have no symbolic program
            continue
        b = {p: int(v) for p, v in c["binding"].items()}
        pts = max(1, int(c["points"]))
        k = 1
        while k < 64 and pts * (k + 1) ** (len(b) + 1) <= 1.5e8:
            k += 1
        if k >= 2:
            out.append((kid, {p: v * k for p, v in b.items()}))
    return out


@pytest.mark.gpu
def test_enumerate_equals_symbolic_on_every_suite_kernel_scaled():
    """GPU brute force == the symbolic programs on every bundled suite kernel
    at scaled bindings (counts bit-exact)."""
    cases = _scaled_cases()
    assert len(cases) >= 50
    for kid, b in cases:
        counts, points = kc.load_enum_program(kid).enumerate_points(b)
        assert counts == _symbolic_counts(kid, b), (kid, b)


def _fd_kernels():
    return [k for k in load_golden("enum_fd.json")["kernels"] if "cases" in k]


def test_floordiv_domain_kernels_parse():
    ks = _fd_kernels()
    assert len(ks) == 60
    for k in ks:
        kc.EnumProgram(k["enum_text"])


@pytest.mark.gpu
def test_enumerate_floordiv_over_domain_variables_matches_reference():
    """60 random kernels whose loop bounds divide domain variables
    (tests/gen/gen_enum_fd_kernels.py: `j = i // 3 .. (i + 1) // 2 + 1`,
    `(i + n) // 3 + 1`, ...), which the reference walks with its generic
    Walker (enumerate.cpp:31-90): counts, visited points and errors equal
    its enumerate_points (tests/golden/enum_fd.json), and the domain walk
    runs on the GPU (floor-division terms KeFd of the rows)."""
    n_ok = 0
    for k in _fd_kernels():
        p = kc.EnumProgram(k["enum_text"])
        for c in k["cases"]:
            b = {q: int(v) for q, v in c["binding"].items()}
            if c["status"] != "ok":
                with pytest.raises(kc.KcgError) as e:
                    p.enumerate_points(b)
                assert e.value.name == c["status"], (k["id"], b)
                continue
            counts, points = p.enumerate_points(b)
            want = {key: int(v) for key, v in c["counts"].items()}
            assert counts == want, (k["id"], b, counts, want)
            assert points == int(c["points"]), (k["id"], b, points, c["points"])
            n_ok += 1
    assert n_ok > 900


GUARDED_FD = """kernelcost-enum v1
kernel x_fdg
param n
assume n >= 1
array a global 32 2 1
array o global 32 2 1
group (n)//2
stmt assign
var g0 0 | (n)//2
var l0 0 | 4
var i 0 | n
var j 0 | (i)//2 + 1
var k (j)//3 | (j + 1)//2 + 1
guard i + l0 < n
access o store 0 | j + 2*k | 3*j + 1
access a load 0 | 3*k + 1 | g0 + 2*j
op flop.f32.addsub 1
op flop.f32.mul 2
endstmt
end
"""


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 5, 8, 13])
def test_enumerate_floordiv_with_guards_brute_force(n):
    """A guarded statement with floordiv-over-domain loop bounds, the case
    the reference's enumerate_points gets wrong (its FastDomain constructor
    returns from the guard loop after a bound failed to compile with ok
    still true and incomplete rows: 0 points, enumerate.cpp:204-214; see
    DESIGN.md 4b) -- against a direct walk of the same domain with the
    reference Walker's rules (a failing guard is one visited dead end)."""
    leaves = visited = 0
    for g0 in range(n // 2):
        for l0 in range(4):
            for i in range(n):
                if not i + l0 < n:
                    visited += 1
                    continue
                for j in range(0, i // 2 + 1):
                    for k in range(j // 3, (j + 1) // 2 + 1):
                        leaves += 1
                        visited += 1
    counts, points = kc.EnumProgram(GUARDED_FD).enumerate_points({"n": n})
    assert points == visited
    assert counts.get("flop.f32.addsub", 0) == leaves and counts.get("flop.f32.mul", 0) == 2 * leaves
