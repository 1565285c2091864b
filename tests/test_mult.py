"""General multiplication operators (SPEC.md:396-399 MultOperator{A, B, apply},
SPEC.md:424-432 builtin_mult_product(A)): the oracle's residue loop with
A inputs and B outputs, checked against direct linear convolutions, and the GPU path against the
oracle on the same seeded inputs (marked gpu)."""
import numpy as np
import pytest

from oracle_lib import rel_l2


def _rand(rng, n):
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


def _lin(f, g, L):
    return np.convolve(f, g)[:L]


def _pairs(blocks, real):
    """A = 2 -> B = 3: F0 F0, F0 F1, F1 F1 (the quadratic products of a 2-component field)."""
    f0, f1 = blocks[0].copy(), blocks[1].copy()
    blocks[0][:] = f0 * f0
    blocks[1][:] = f0 * f1
    blocks[2][:] = f1 * f1


# ------------------------------------------------------------------ oracle (CPU) --
def test_callback_product_equals_builtin(oracle):
    rng = np.random.default_rng(1)
    for L, M, m, sym in [(6, 11, 4, 0), (12, 23, 5, 0), (17, 33, 17, 0), (15, 22, 8, 1), (15, 22, 8, 2), (31, 46, 8, 2)]:
        f, g = _rand(rng, (L + 1) // 2 if sym == 2 else L), _rand(rng, (L + 1) // 2 if sym == 2 else L)
        if sym == 2:
            f[0], g[0] = f[0].real, g[0].real

        def prod(b, real):
            b[0] *= b[1]

        h = oracle.convolve_general([(L, M, m, sym)], [f, g], 1, prod)[0]
        ref = oracle.convolve([(L, M, m, sym)], f, g)
        assert rel_l2(h, ref) < 1e-15, (L, M, m, sym)


def test_builtin_product_three_inputs(oracle):
    """builtin_mult_product(3): f * g * k, alias-free for M >= 3L - 2."""
    rng = np.random.default_rng(2)
    for L, m in [(8, 4), (8, 22), (13, 6), (20, 7)]:
        M = 3 * L - 2
        f, g, k = (_rand(rng, L) for _ in range(3))
        h = oracle.convolve_general([(L, M, m, 0)], [f, g, k], 1)[0]
        ref = np.convolve(np.convolve(f, g), k)[:L]
        assert rel_l2(h, ref) < 1e-13, (L, m)


def test_two_to_three_operator(oracle):
    rng = np.random.default_rng(3)
    for L, M, m in [(10, 19, 4), (10, 19, 10), (16, 31, 6), (9, 17, 2)]:
        f, g = _rand(rng, L), _rand(rng, L)
        hs = oracle.convolve_general([(L, M, m, 0)], [f, g], 3, _pairs)
        for h, ref in zip(hs, [_lin(f, f, L), _lin(f, g, L), _lin(g, g, L)]):
            assert rel_l2(h, ref) < 1e-13, (L, M, m)


def test_one_to_one_operator_and_hermitian_real_blocks(oracle):
    """A = 1: F -> F F (a self-convolution); Hermitian residues reach the operator as float64."""
    rng = np.random.default_rng(4)
    seen = []

    def square(b, real):
        seen.append((b[0].dtype, real))
        b[0] *= b[0]

    for L, M, m, sym in [(11, 21, 4, 0), (15, 22, 8, 2), (15, 22, 4, 2)]:
        f = _rand(rng, (L + 1) // 2 if sym == 2 else L)
        if sym == 2:
            f[0] = f[0].real
        h = oracle.convolve_general([(L, M, m, sym)], [f], 1, square)[0]
        ref = oracle.convolve([(L, M, m, sym)], f, f)
        assert rel_l2(h, ref) < 1e-14
    assert (np.dtype(np.float64), True) in seen and (np.dtype(np.complex128), False) in seen


def test_nd_general_operator(oracle):
    """2D complex and 3D Hermitian with A = 2 -> B = 3 against three binary convolutions."""
    rng = np.random.default_rng(5)
    for axes, shape in [([(6, 11, 4, 0), (5, 9, 3, 0)], (6, 5)),
                        ([(5, 8, 3, 1), (7, 11, 4, 1), (7, 11, 4, 2)], (5, 7, 4))]:
        f, g = _rand(rng, shape), _rand(rng, shape)
        if axes[-1][3] == 2:
            Ls = [a[0] for a in axes]
            f, g = oracle.symmetrize(Ls, f), oracle.symmetrize(Ls, g)
        hs = oracle.convolve_general(axes, [f, g], 3, _pairs)
        for h, (x, y) in zip(hs, [(f, f), (f, g), (g, g)]):
            assert rel_l2(h, oracle.convolve(axes, x, y)) < 1e-13


def test_operator_errors(oracle):
    import ctypes as C

    from paper_2303_17510_b200 import _abi

    def bad(b, real):
        raise RuntimeError("operator failure")

    with pytest.raises(ValueError, match="callback"):
        oracle.convolve_general([(8, 16, 8, 0)], [np.ones(8, complex)], 1, bad)
    with pytest.raises(ValueError):  # builtin product needs A >= 2
        oracle.convolve_general([(8, 16, 8, 0)], [np.ones(8, complex)], 1)
    d = _abi.Desc()
    d.dims, d.A, d.B, d.mult = 1, 2, 1, _abi.MULT_CALLBACK
    d.axis[0] = _abi.Axis(8, 16, 8, 0)
    h = C.c_void_p()
    assert oracle.lib.hconv_plan_create(C.byref(d), C.byref(h)) == _abi.INVALID_ARG  # no mult_fn


# ------------------------------------------------------------------- GPU parity --
@pytest.mark.gpu
@pytest.mark.parametrize("L,M,m,sym,C_", [(1024, 2047, 1024, 0, 9), (6000, 11999, 1536, 0, 5), (6000, 11999, 6144, 0, 3),
                                          (511, 766, 256, 2, 7), (1023, 1534, 256, 2, 4), (511, 766, 128, 1, 6)])
def test_gpu_general_operator_1d(cuda, oracle, L, M, m, sym, C_):
    import torch

    rng = np.random.default_rng(L + m)
    S = (L + 1) // 2 if sym == 2 else L
    f, g = _rand(rng, (C_, S)), _rand(rng, (C_, S))
    if sym == 2:
        f[:, 0], g[:, 0] = f[:, 0].real, g[:, 0].real

    def pairs_t(b, real):
        f0, f1 = b[0].clone(), b[1].clone()
        b[0].copy_(f0 * f0)
        b[1].copy_(f0 * f1)
        b[2].copy_(f1 * f1)

    op = cuda.mult_operator(2, 3, pairs_t)
    plan = cuda.Conv1dPlan(L, M, m, cuda.Symmetry(sym), op, C_=C_)
    ft, gt = torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()
    outs = [torch.empty_like(ft) for _ in range(3)]
    cuda.convolve([ft, gt], op, plan, out=outs)
    torch.cuda.synchronize()
    refs = oracle.convolve_general([(L, M, m, sym)], [f, g], 3, _pairs, C_=C_)
    for o, r in zip(outs, refs):
        assert rel_l2(o.cpu().numpy(), r) <= 1e-12
    # builtin product with three inputs (general loop on the device)
    k = _rand(rng, (C_, S))
    if sym == 2:
        k[:, 0] = k[:, 0].real
    op3 = cuda.builtin_mult_product(3)
    plan3 = cuda.Conv1dPlan(L, M, m, cuda.Symmetry(sym), op3, C_=C_)
    h = cuda.convolve([ft, gt, torch.from_numpy(k).cuda()], op3, plan3, out=torch.empty_like(ft))[0]
    ref = oracle.convolve_general([(L, M, m, sym)], [f, g, k], 1, C_=C_)[0]
    assert rel_l2(h.cpu().numpy(), ref) <= 1e-12
    # in place (outputs overwrite the first B inputs) and through the host-buffer entry point
    fh, gh = torch.from_numpy(f.copy()), torch.from_numpy(g.copy())
    hb = cuda.convolve_host([fh, gh], op, plan, out=[fh, gh, torch.empty_like(fh)])
    for o, r in zip(hb, refs):
        assert rel_l2(o.numpy(), r) <= 1e-12


@pytest.mark.gpu
def test_gpu_general_operator_nd(cuda, oracle):
    import torch

    rng = np.random.default_rng(9)
    for axes in ([(64, 127, 64, 0), (48, 95, 32, 0)], [(31, 46, 16, 1), (31, 46, 16, 1), (31, 46, 16, 2)]):
        shape = tuple((a[0] + 1) // 2 if a[3] == 2 else a[0] for a in axes)
        f, g = _rand(rng, shape), _rand(rng, shape)
        if axes[-1][3] == 2:
            f, g = oracle.symmetrize([a[0] for a in axes], f), oracle.symmetrize([a[0] for a in axes], g)

        def pairs_t(b, real):
            f0, f1 = b[0].clone(), b[1].clone()
            b[0].copy_(f0 * f0)
            b[1].copy_(f0 * f1)
            b[2].copy_(f1 * f1)

        op = cuda.mult_operator(2, 3, pairs_t)
        plan = cuda.ConvPlanND([cuda.AxisSpec(L, M, m, cuda.Symmetry(s)) for L, M, m, s in axes], op)
        ft, gt = torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()
        outs = cuda.convolve_nd([ft, gt], op, plan, out=[torch.empty_like(ft) for _ in range(3)])
        torch.cuda.synchronize()
        refs = oracle.convolve_general(axes, [f, g], 3, _pairs)
        for o, r in zip(outs, refs):
            assert rel_l2(o.cpu().numpy(), r) <= 1e-12


@pytest.mark.gpu
def test_gpu_operator_stream_order_repeated(cuda, oracle):
    """Repeated calls (no allocation in between, so nothing synchronises by accident): the
    Python operator must run on the library's stream -- NULL is the legacy default stream, not
    a fresh pool stream -- and the native example operator (hconv_example_mult) likewise."""
    import torch

    from paper_2303_17510_b200 import _abi

    rng = np.random.default_rng(12)
    axes = [(31, 46, 16, 1), (31, 46, 16, 1), (31, 46, 16, 2)]
    f, g = _rand(rng, (31, 31, 16)), _rand(rng, (31, 31, 16))
    f, g = oracle.symmetrize([a[0] for a in axes], f), oracle.symmetrize([a[0] for a in axes], g)
    refs = oracle.convolve_general(axes, [f, g], 3, _pairs)

    def pairs_t(b, real):
        f0, f1 = b[0].clone(), b[1].clone()
        b[0].copy_(f0 * f0)
        b[1].copy_(f0 * f1)
        b[2].copy_(f1 * f1)

    ops = [cuda.mult_operator(2, 3, pairs_t), cuda.MultOperator(2, 3, _abi.MULT_CALLBACK, fn=cuda.lib().hconv_example_mult(0))]
    ft, gt = torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()
    for op in ops:
        plan = cuda.ConvPlanND([cuda.AxisSpec(L, M, m, cuda.Symmetry(s)) for L, M, m, s in axes], op)
        outs = [torch.empty_like(ft) for _ in range(3)]
        for _ in range(6):
            cuda.convolve_nd([ft, gt], op, plan, out=outs)
            torch.cuda.synchronize()
            for o, r in zip(outs, refs):
                assert rel_l2(o.cpu().numpy(), r) <= 1e-12
