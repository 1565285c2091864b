"""The CPU oracle pinned to the reference: SPEC known-answer examples (tests/golden/spec_kats.json)
and the SPEC acceptance properties at reduced grids.  The oracle is the
checker of every GPU parity test, so it is tested here first."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import rel_l2

KATS = json.loads((Path(__file__).resolve().parent / "golden" / "spec_kats.json").read_text())


def c(a):
    return np.array([complex(x, y) for x, y in a])


def test_kat_dft(oracle):
    for e in KATS["dft"]:
        np.testing.assert_allclose(oracle.dft(c(e["x"]), e["sign"]), c(e["y"]), atol=1e-15)
    x = np.full(6, 2 + 1j)
    y = oracle.dft(x)
    assert abs(y[0] - 6 * (2 + 1j)) < 1e-12 and np.abs(y[1:]).max() < 1e-12
    rng = np.random.default_rng(0)
    x = rng.standard_normal(8) + 1j * rng.standard_normal(8)
    np.testing.assert_allclose(oracle.dft(oracle.dft(x, 1), -1), 8 * x, atol=1e-12)
    for n in (6, 12, 45, 64, 6144):
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        ref = np.fft.ifft(x) * n  # numpy's inverse has the + sign of the paper's forward
        assert rel_l2(oracle.dft(x, 1, naive=False), ref) < 1e-14


def test_kat_forward(oracle):
    for e in KATS["forward"]:
        L, M, m = e["LMm"]
        p = oracle.derive(L, M, m, e["sym"])
        F = oracle.forward(p, c(e["f"]), e["r"])
        np.testing.assert_allclose(F, c(e["F"]).real if e["sym"] == 2 else c(e["F"]), atol=1e-13, err_msg=e["src"])


def test_kat_convolve_and_direct(oracle):
    for e in KATS["convolve"]:
        L, M, m = e["LMm"]
        h = oracle.convolve([(L, M, m, e["sym"])], c(e["f"]), c(e["g"]))
        np.testing.assert_allclose(h, c(e["h"]), atol=1e-14, err_msg=e["src"])
    for e in KATS["direct"]:
        full = np.convolve(e["f"], e["g"])
        assert list(full) == e["full"]
        h = oracle.direct([0], [2], np.array(e["f"], complex), np.array(e["g"], complex))
        np.testing.assert_allclose(h, e["window"], atol=1e-14)
        h = oracle.convolve([(2, 3, 2, 0)], np.array(e["f"], complex), np.array(e["g"], complex))
        np.testing.assert_allclose(h, e["window"], atol=1e-14)
    # delta * g = g
    g = np.arange(8) + 1j
    d = np.zeros(8, complex)
    d[0] = 1
    np.testing.assert_allclose(oracle.convolve([(8, 16, 8, 0)], d, g), g, atol=1e-13)


def test_kat_slice_indices(oracle):
    e = KATS["slice_indices"][0]
    p = oracle.derive(e["L"], e["M"], e["m"], 0)
    rng = np.random.default_rng(1)
    f = rng.standard_normal(e["L"]) + 1j * rng.standard_normal(e["L"])
    full = np.fft.ifft(np.concatenate([f, np.zeros(p.q * p.m - e["L"])])) * p.q * p.m
    np.testing.assert_allclose(oracle.slice(p, f, e["r"]), full[e["k"]], atol=1e-13)


@pytest.mark.parametrize("sym", [0, 1, 2])
def test_spectral_slicing_and_roundtrip(oracle, sym):
    """SPEC acceptance 2 and 3 (L <= 24, M in {2L-1, 2L, 3L}, every valid m)."""
    rng = np.random.default_rng(sym)
    for L in range(1, 25):
        if sym == 2 and L % 2 == 0:
            continue
        for M in sorted({max(L, 2 * L - 1), 2 * L, 3 * L}):
            for m in range(1, M + 1):
                p = oracle.derive(L, M, m, sym)
                S = oracle.data_length(p)
                f = rng.standard_normal(S) + 1j * rng.standard_normal(S)
                if sym == 2:
                    f[0] = f[0].real
                acc = np.zeros(S, complex)
                for r in range(p.n):
                    F = oracle.forward(p, f, r)
                    G = oracle.slice(p, f, r)
                    assert rel_l2(F, G) <= 1e-12, (L, M, m, r)
                    acc += oracle.backward(p, F, r)
                assert rel_l2(acc, p.q * p.m * f) <= 1e-11, (L, M, m)


def test_conv1d_oracle_equivalence(oracle):
    """SPEC acceptance 4: complex L <= 48 (M in {2L-1, 2L}), centered/Hermitian L <= 31, 3 seeds."""
    for seed in (1, 2, 3):
        rng = np.random.default_rng(seed)
        for L in range(1, 49, 3):
            for M in (max(L, 2 * L - 1), 2 * L):
                for m in sorted({1, 2, max(1, L // 4), L, M}):
                    f = rng.uniform(-1, 1, L) + 1j * rng.uniform(-1, 1, L)
                    g = rng.uniform(-1, 1, L) + 1j * rng.uniform(-1, 1, L)
                    h = oracle.convolve([(L, M, m, 0)], f, g)
                    assert rel_l2(h, np.convolve(f, g)[:L]) <= 1e-11
        for sym in (1, 2):
            for L in range(1, 32, 2):
                M = (3 * L + 1) // 2
                S = (L + 1) // 2 if sym == 2 else L
                for m in sorted({1, 2, max(1, L // 3), L}):
                    f = rng.uniform(-1, 1, S) + 1j * rng.uniform(-1, 1, S)
                    g = rng.uniform(-1, 1, S) + 1j * rng.uniform(-1, 1, S)
                    if sym == 2:
                        f[0], g[0] = f[0].real, g[0].real
                    h = oracle.convolve([(L, M, m, sym)], f, g)
                    assert rel_l2(h, oracle.direct([sym], [L], f, g)) <= 1e-11, (sym, L, m)


def test_padding_length_independence(oracle):
    """SPEC acceptance 5: L = 17, M in {33, 34, 40, 64}."""
    rng = np.random.default_rng(4)
    f = rng.uniform(-1, 1, 17) + 1j * rng.uniform(-1, 1, 17)
    g = rng.uniform(-1, 1, 17) + 1j * rng.uniform(-1, 1, 17)
    outs = [oracle.convolve([(17, M, m, 0)], f, g) for M in (33, 34, 40, 64) for m in (5, 17, M)]
    for o in outs[1:]:
        assert rel_l2(o, outs[0]) <= 1e-11


def test_nd_oracle(oracle):
    """SPEC acceptance 6 (reduced): 2D complex L <= 12, 3D complex L <= 6, 2D Hermitian L <= 9."""
    rng = np.random.default_rng(6)
    for L in (3, 8, 12):
        f = rng.uniform(-1, 1, (L, L)) + 1j * rng.uniform(-1, 1, (L, L))
        g = rng.uniform(-1, 1, (L, L)) + 1j * rng.uniform(-1, 1, (L, L))
        h = oracle.convolve([(L, 2 * L, max(1, L // 2), 0), (L, 2 * L, L, 0)], f, g)
        assert rel_l2(h, oracle.direct([0, 0], [L, L], f, g)) <= 1e-11
    L = 6
    f = rng.uniform(-1, 1, (L, L, L)) + 1j * rng.uniform(-1, 1, (L, L, L))
    g = rng.uniform(-1, 1, (L, L, L)) + 1j * rng.uniform(-1, 1, (L, L, L))
    h = oracle.convolve([(L, 2 * L, 3, 0)] * 3, f, g)
    assert rel_l2(h, oracle.direct([0, 0, 0], [L] * 3, f, g)) <= 1e-11
    for L in (5, 9):
        M = (3 * L + 1) // 2
        sh = (L, (L + 1) // 2)
        f = oracle.symmetrize([L, L], rng.uniform(-1, 1, sh) + 1j * rng.uniform(-1, 1, sh))
        g = oracle.symmetrize([L, L], rng.uniform(-1, 1, sh) + 1j * rng.uniform(-1, 1, sh))
        h = oracle.convolve([(L, M, 2, 1), (L, M, 3, 2)], f, g)
        assert rel_l2(h, oracle.direct([1, 2], [L, L], f, g)) <= 1e-11


def test_conjugate_pair(oracle):
    """SPEC acceptance 8: forward_conjugate_pair against independent forwards / the naive slice."""
    rng = np.random.default_rng(8)
    for L, M, m in [(12, 36, 3), (10, 30, 2), (20, 61, 4), (9, 40, 3)]:
        p = oracle.derive(L, M, m, 0)
        if p.n < 3:
            continue
        f = rng.standard_normal(L) + 1j * rng.standard_normal(L)
        qm = p.q * p.m
        full = np.fft.ifft(np.concatenate([f, np.zeros(qm - L)])) * qm
        for v in range(1, p.n):
            if 2 * v == p.n:
                continue
            a, b = oracle.conjugate_pair(p, f, v)
            np.testing.assert_allclose(a, oracle.forward(p, f, v), atol=1e-13)
            ks = [(p.q * l + u * p.n - v) % qm for u in range(p.p) for l in range(p.m)]
            np.testing.assert_allclose(b, full[ks], atol=1e-12)


def test_symmetrize_boundary(oracle):
    rng = np.random.default_rng(9)
    L = 7
    f = rng.standard_normal((L, L, 4)) + 1j * rng.standard_normal((L, L, 4))
    s = oracle.symmetrize([L, L, L], f.copy())
    H = L // 2
    for x in range(L):
        for y in range(L):
            assert s[x, y, 0] == np.conj(s[2 * H - x, 2 * H - y, 0])
    np.testing.assert_array_equal(oracle.symmetrize([L, L, L], s.copy()), s)  # idempotent
