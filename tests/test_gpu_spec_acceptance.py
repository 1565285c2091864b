"""SPEC.md acceptance criteria on the sm_100a path, through the C ABI.

The oracle's own acceptance tests (tests/test_oracle.py) pin the CPU restatement; these run the
same grids on the GPU kernels and compare with the oracle / naive references:
  2  complex spectral slicing, L <= 24, M in {2L-1, 2L, 3L}, every valid m (all three kinds)
  3  roundtrip completeness sum_r backward(forward(f, r), r) = qm f
  4  1D convolution vs direct sums (complex L <= 48, centered / Hermitian L <= 31, 3 seeds)
  5  padding-length independence (L = 17, M in {33, 34, 40, 64})
  6  N-D vs brute force (2D complex L <= 12, 3D complex L <= 6, 2D Hermitian L <= 9)
  8  conjugate pair = two independent forwards, 50 random configurations with n >= 3
  9  performance smoke: tuned 3D L=80 M=160 no slower than explicit next-power-of-two padding;
     L=64 M=128 within 1.15 of the best explicit plan
(1 and 7 are in tests/test_plan.py and test_gpu_parity.py::test_work_memory_bound; 10, the
tuner, in test_gpu_parity.py::test_planner_*.)"""
import numpy as np
import pytest

from oracle_lib import rel_l2

pytestmark = pytest.mark.gpu


def _t(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _rand(rng, shape):
    return rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)


@pytest.mark.parametrize("sym", [0, 1, 2])
def test_spectral_slicing_and_roundtrip(cuda, oracle, sym):
    """criteria 2 and 3: every residue block (reference order) against the naive padded-DFT
    slice within 1e-12, and the unnormalised roundtrip qm f within 1e-11, over the whole grid."""
    rng = np.random.default_rng(10 + sym)
    cases = 0
    for L in range(1, 25):
        if sym == 2 and L % 2 == 0:
            continue
        for M in sorted({max(L, 2 * L - 1), 2 * L, 3 * L}):
            for m in range(1, M + 1):
                try:
                    pp = cuda.deriveParams(L, M, m, cuda.Symmetry(sym))
                except ValueError:
                    continue
                op = oracle.derive(L, M, m, sym)
                S = pp.dataLength()
                f = _rand(rng, (1, S))
                if sym == 2:
                    f[:, 0] = f[:, 0].real
                acc = None
                for r in range(pp.n):
                    F = cuda.forward(_t(f), pp, r)
                    assert rel_l2(F.cpu().numpy()[0], oracle.slice(op, f[0], r)) <= 1e-12, (L, M, m, r)
                    acc = cuda.backward(F, pp, r, h=acc, accumulate=acc is not None)
                assert rel_l2(acc.cpu().numpy()[0], pp.q * pp.m * f[0]) <= 1e-11, (L, M, m)
                cases += 1
    assert cases > 500


def test_conv1d_vs_direct_sums(cuda, oracle):
    """criterion 4: hybrid 1D convolutions equal the direct sums within 1e-11, 3 seeds."""
    for seed in (1, 2, 3):
        rng = np.random.default_rng(seed)
        for L in range(1, 49, 3):
            for M in (max(L, 2 * L - 1), 2 * L):
                for m in sorted({1, 2, max(1, L // 4), L, M}):
                    f, g = _rand(rng, (2, L)), _rand(rng, (2, L))
                    plan = cuda.Conv1dPlan(L, M, m, C_=2)
                    h = cuda.convolve([_t(f), _t(g)], plan.mult, plan, out=_t(f) * 0)[0].cpu().numpy()
                    for c in range(2):
                        assert rel_l2(h[c], np.convolve(f[c], g[c])[:L]) <= 1e-11, (L, M, m)
        for sym in (1, 2):
            for L in range(1, 32, 2):
                M = (3 * L + 1) // 2
                S = (L + 1) // 2 if sym == 2 else L
                for m in sorted({1, 2, max(1, L // 3), L}):
                    f, g = _rand(rng, (1, S)), _rand(rng, (1, S))
                    if sym == 2:
                        f[:, 0], g[:, 0] = f[:, 0].real, g[:, 0].real
                    plan = cuda.Conv1dPlan(L, M, m, cuda.Symmetry(sym))
                    h = cuda.convolve([_t(f), _t(g)], plan.mult, plan, out=_t(f) * 0)[0].cpu().numpy()[0]
                    assert rel_l2(h, oracle.direct([sym], [L], f[0], g[0])) <= 1e-11, (sym, L, m)


def test_padding_length_independence(cuda):
    """criterion 5: L = 17, M in {33, 34, 40, 64}, several m -- results agree within 1e-11."""
    rng = np.random.default_rng(5)
    f, g = _rand(rng, (1, 17)), _rand(rng, (1, 17))
    outs = []
    for M in (33, 34, 40, 64):
        for m in (5, 17, M):
            plan = cuda.Conv1dPlan(17, M, m)
            outs.append(cuda.convolve([_t(f), _t(g)], plan.mult, plan, out=_t(f) * 0)[0].cpu().numpy())
    for o in outs[1:]:
        assert rel_l2(o, outs[0]) <= 1e-11


def test_nd_vs_brute_force(cuda, oracle):
    """criterion 6: 2D complex L <= 12, 3D complex L <= 6, 2D Hermitian L <= 9 vs direct sums."""
    import torch

    rng = np.random.default_rng(6)
    for L in (3, 8, 12):
        f, g = _rand(rng, (L, L)), _rand(rng, (L, L))
        plan = cuda.ConvPlanND([cuda.AxisSpec(L, 2 * L, max(1, L // 2)), cuda.AxisSpec(L, 2 * L, L)])
        h = cuda.convolve_nd([_t(f), _t(g)], plan.mult, plan, out=torch.empty((L, L), dtype=torch.complex128,
                                                                                 device="cuda"))[0]
        assert rel_l2(h.cpu().numpy(), oracle.direct([0, 0], [L, L], f, g)) <= 1e-11
    L = 6
    f, g = _rand(rng, (L, L, L)), _rand(rng, (L, L, L))
    plan = cuda.ConvPlanND([cuda.AxisSpec(L, 2 * L, 3)] * 3)
    h = cuda.convolve_nd([_t(f), _t(g)], plan.mult, plan, out=_t(f) * 0)[0]
    assert rel_l2(h.cpu().numpy(), oracle.direct([0, 0, 0], [L] * 3, f, g)) <= 1e-11
    for L in (5, 9):
        M = (3 * L + 1) // 2
        sh = (L, (L + 1) // 2)
        f = oracle.symmetrize([L, L], _rand(rng, sh))
        g = oracle.symmetrize([L, L], _rand(rng, sh))
        plan = cuda.ConvPlanND([cuda.AxisSpec(L, M, 2, cuda.Symmetry.Centered),
                                cuda.AxisSpec(L, M, 3, cuda.Symmetry.Hermitian)])
        h = cuda.convolve_nd([_t(f), _t(g)], plan.mult, plan, out=_t(f) * 0)[0]
        assert rel_l2(h.cpu().numpy(), oracle.direct([1, 2], [L, L], f, g)) <= 1e-11


def test_conjugate_pair_50_configurations(cuda):
    """criterion 8: forward_conjugate_pair equals two independent forward calls within 1e-13
    (relative) across 50 random configurations with n >= 3."""
    rng = np.random.default_rng(8)
    done = 0
    while done < 50:
        L = int(rng.integers(2, 200))
        M = int(rng.integers(L, 4 * L + 1))
        m = int(rng.integers(1, max(2, L // 2)))
        pp = cuda.deriveParams(L, M, m)
        if pp.n < 3:
            continue
        v = int(rng.integers(1, pp.n))
        if 2 * v == pp.n:
            continue
        f = _rand(rng, (2, L))
        Fv, Fn = cuda.forward_conjugate_pair(_t(f), pp, v)
        ref_v = cuda.forward(_t(f), pp, v).cpu().numpy()
        ref_n = cuda.forward(_t(f), pp, pp.n - v).cpu().numpy()
        assert rel_l2(Fv.cpu().numpy(), ref_v) <= 1e-13
        # F_{q l + u n - v} = F_{(n - v) + n (k' - 1)}: block n - v one natural index back; the
        # reference order puts natural k' at (k' % pe) m + k' / pe (pe = p for inner blocks)
        B = pp.blockLength()
        pe = pp.p if (pp.p > 2 and B == pp.p * pp.m) else 1
        kk = np.arange(B)
        ref_pos = (kk % pe) * pp.m + kk // pe

        def nat(x):
            return x[:, ref_pos]

        Fn = nat(Fn.cpu().numpy())
        shifted = np.roll(nat(ref_n), 1, axis=1)
        assert rel_l2(Fn, shifted) <= 1e-13, (L, M, m, v)
        done += 1


def _timed(fn, reps=7):
    import torch

    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def test_performance_smoke(cuda):
    """criterion 9 (record-and-report): the device-tuned 3D L=80 M=160 plan is no slower than
    explicit next-power-of-two padding, and at L=64 M=128 it is within 1.15 of the best explicit
    plan (timed on the device, medians of 5)."""
    import torch

    res = {}
    for L, M, explicit in ((80, 160, [256]), (64, 128, [128, 256])):
        f = torch.empty((L, L, L), dtype=torch.complex128, device="cuda")
        g = torch.empty_like(f)
        o = torch.empty_like(f)
        cuda.fill_uniform(f, 9, 0)
        cuda.fill_uniform(g, 9, 1)
        tuned = cuda.ConvPlanND([cuda.AxisSpec(L, M, None)] * 3)
        t_tuned = _timed(lambda: cuda.convolve_nd([f, g], tuned.mult, tuned, out=o))
        t_expl = []
        for m in explicit:
            pl = cuda.ConvPlanND([cuda.AxisSpec(L, M, m)] * 3)
            t_expl.append(_timed(lambda: cuda.convolve_nd([f, g], pl.mult, pl, out=o)))
        res[(L, M)] = (t_tuned, t_expl, [p.m for p in tuned.params])
    t, te, ms = res[(80, 160)]
    # when the tuner picks the power of two itself the two timings are the same plan: allow 5 %
    # run-to-run noise (SPEC.md:693 makes this a record-and-report check, not a correctness one)
    assert t <= 1.0 * te[0] * 1.05, res
    t, te, ms = res[(64, 128)]
    assert t <= 1.15 * min(te), res
    print("performance smoke", res)
