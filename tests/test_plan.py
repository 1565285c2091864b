"""Plan module (the reference's only compiled code): the product's host plan (through the CUDA
library's C ABI, no GPU needed) and the oracle's restatement, pinned to the reference's own
plan.cpp -- live via oracle/_ref when it is built, and via tests/golden/plan_ref.json."""
import ctypes as C
import json
import math
from pathlib import Path

import pytest

from paper_2303_17510_b200 import _abi

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def cuda_lib():
    from paper_2303_17510_b200 import hconv

    return hconv.lib()


def _derive(lib, L, M, m, s):
    p = _abi.Params()
    st = lib.hconv_derive_params(L, M, m, s, C.byref(p))
    return st, p


def _row(lib, L, M, m, s):
    st, p = _derive(lib, L, M, m, s)
    assert st == 0
    return [p.L, p.M, p.m, p.p, p.q, p.n, p.D, p.C, p.S, p.inplace, p.symmetry, p.regime,
            lib.hconv_block_length(C.byref(p)), lib.hconv_stored_length(C.byref(p)), lib.hconv_padded_length(C.byref(p))]


@pytest.mark.parametrize("which", ["cuda", "oracle"])
def test_plan_matches_reference_fixture(which, cuda_lib, oracle):
    lib = cuda_lib if which == "cuda" else oracle.lib
    rows = json.loads((GOLD / "plan_ref.json").read_text())["rows"]
    for r in rows:
        L, M, m, s = r[:4]
        assert _row(lib, L, M, m, s) == r[4:], (which, r[:4])


def test_plan_matches_live_reference_full_grid(cuda_lib, oracle, ref_plan):
    """SPEC acceptance 1: 1 <= L <= M <= 64, 1 <= m <= 64, every symmetry."""
    out = (C.c_uint64 * 12)()
    for s in (0, 1, 2):
        for L in range(1, 65):
            for M in range(L, 65):
                for m in range(1, 65):
                    assert ref_plan.ref_derive_params(L, M, m, s, out) == 0
                    want = list(out)
                    st, p = _derive(cuda_lib, L, M, m, s)
                    got = [p.L, p.M, p.m, p.p, p.q, p.n, p.D, p.C, p.S, p.inplace, p.symmetry, p.regime]
                    assert got == want, (L, M, m, s)
                    # invariants: pm >= L, qm >= M, (p-1)m < L, centered p even
                    assert p.p * m >= L and p.q * m >= M
                    if s == 0:
                        assert (p.p - 1) * m < L
                    else:
                        assert p.p % 2 == 0
    for L, M, m in [(0, 4, 2), (5, 4, 2), (5, 8, 0)]:
        assert ref_plan.ref_derive_params(L, M, m, 0, out) == 1
        assert _derive(cuda_lib, L, M, m, 0)[0] == _abi.INVALID_ARG
        assert _derive(oracle.lib, L, M, m, 0)[0] == _abi.INVALID_ARG


def test_root_and_tables_vs_reference(cuda_lib, ref_plan):
    re, im = C.c_double(), C.c_double()
    rr, ri = C.c_double(), C.c_double()
    for N in (1, 2, 3, 4, 12, 768, 2048, 12288, 24576):
        for k in list(range(-3, 20)) + [N - 1, N, N + 5, 7 * N + 3, -N - 2]:
            assert cuda_lib.hconv_root(N, k, C.byref(re), C.byref(im)) == 0
            assert ref_plan.ref_root(N, k, C.byref(rr), C.byref(ri)) == 0
            assert abs(re.value - rr.value) <= 1e-15 and abs(im.value - ri.value) <= 1e-15
    assert cuda_lib.hconv_root(0, 1, C.byref(re), C.byref(im)) == _abi.INVALID_ARG
    for N in (5, 64, 3072):
        t = (C.c_double * (2 * N))()
        assert cuda_lib.hconv_root_table(N, C.cast(t, C.c_void_p)) == 0
        r = (C.c_double * (2 * N))()
        assert ref_plan.ref_root_table(N, 0, N, r) == 0
        # the reference accumulates step*k in double (plan.cpp:96-98); ours reduces k exactly first
        assert max(abs(t[i] - r[i]) for i in range(2 * N)) <= 1e-14
        # group law within 1e-14
        z = [complex(t[2 * i], t[2 * i + 1]) for i in range(N)]
        for a, b in [(1, 2), (N // 2, N - 1), (3 % N, 5 % N)]:
            assert abs(z[a] * z[b] - z[(a + b) % N]) <= 1e-14
    assert ref_plan.ref_root_table_at(12, 5, 7, C.byref(rr), C.byref(ri)) == 0


def test_work_memory_vs_reference(cuda_lib, ref_plan):
    iw, ew = C.c_uint64(), C.c_double()
    riw, rew = C.c_uint64(), C.c_double()
    for (L, M, m, s) in [(8, 16, 8, 0), (64, 128, 64, 0), (64, 128, 16, 0), (511, 766, 256, 1), (16383, 24574, 8192, 2)]:
        for A, B, d in [(2, 1, 1), (2, 1, 2), (3, 5, 3), (6, 8, 2)]:
            _, p = _derive(cuda_lib, L, M, m, s)
            assert cuda_lib.hconv_work_memory_words(C.byref(p), A, B, d, L, C.byref(iw), C.byref(ew)) == 0
            assert ref_plan.ref_work_memory_words(L, M, m, s, A, B, d, L, C.byref(riw), C.byref(rew)) == 0
            assert iw.value == riw.value and ew.value == pytest.approx(rew.value, rel=1e-15)
    _, p = _derive(cuda_lib, 8, 16, 8, 0)
    assert cuda_lib.hconv_work_memory_words(C.byref(p), 0, 1, 1, 8, C.byref(iw), C.byref(ew)) == _abi.INVALID_ARG
    assert cuda_lib.hconv_work_memory_words(C.byref(p), 2, 1, 4, 8, C.byref(iw), C.byref(ew)) == _abi.INVALID_ARG


def test_names(cuda_lib, ref_plan):
    s = C.c_int()
    for i, n in enumerate(["complex", "centered", "hermitian"]):
        assert cuda_lib.hconv_symmetry_name(i).decode() == n == ref_plan.ref_symmetry_name(i).decode()
        assert cuda_lib.hconv_symmetry_from_name(n.encode(), C.byref(s)) == 0 and s.value == i
    assert cuda_lib.hconv_symmetry_from_name(b"real", C.byref(s)) == _abi.INVALID_ARG
    assert ref_plan.ref_symmetry_from_name(b"real", C.byref(s)) == 1


def test_spec_kats_plan(cuda_lib):
    k = json.loads((GOLD / "spec_kats.json").read_text())
    for e in k["derive_params"]:
        st, p = _derive(cuda_lib, *e["args"])
        assert st == 0 and p.p == e["p"] and p.q == e["q"], e["src"]
        if "n" in e:
            assert p.n == e["n"], e["src"]
    for e in k["derive_params_errors"]:
        assert _derive(cuda_lib, *e["args"])[0] == _abi.INVALID_ARG, e["src"]
    re, im = C.c_double(), C.c_double()
    for e in k["root"]:
        cuda_lib.hconv_root(e["N"], e["k"], C.byref(re), C.byref(im))
        assert abs(re.value - e["value"][0]) < 1e-15 and abs(im.value - e["value"][1]) < 1e-15, e["src"]
    iw, ew = C.c_uint64(), C.c_double()
    for e in k["work_memory"]:
        _, p = _derive(cuda_lib, *e["LMm"], 0)
        cuda_lib.hconv_work_memory_words(C.byref(p), e["A"], e["B"], e["d"], e["Lw"], C.byref(iw), C.byref(ew))
        if "implicit" in e:
            assert iw.value == e["implicit"] and ew.value == e["explicit"], e["src"]
        else:
            assert iw.value / ew.value == pytest.approx(e["ratio"]), e["src"]
