"""Stress cases of every kernel family (the synchronisation check in place of compute-sanitizer,
which this GPU pool does not allow: runs under it have left GPUs needing a reset).

  HCONV_POISON=1 python tools/stress_cases.py [case ...]

Every scratch / work allocation of the library is NaN-filled (HCONV_POISON=1), so a read
before write (a missing barrier, a TMA copy consumed before its mbarrier phase, a proxy fence
missing between generic stores and bulk reads) shows up as NaN or as a mismatch; each case runs
REPEAT times on fresh outputs and must be bit-identical from run to run (races are
nondeterministic) and within 1e-12 of the CPU oracle."""
import sys
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))
from oracle_lib import Oracle, rel_l2  # noqa: E402
from paper_2303_17510_b200 import hconv  # noqa: E402

# name: (kind, axes [(L, M, m, sym)], copies) -- the kernel each one selects
CASES = {
    "ip_c2": ("1d", [(6000, 11999, 6144, 0)], 301),       # k_conv1d_ip4: persistent loop (> 2 lines per CTA), both residues in flight
    "ip_short": ("1d", [(3100, 9000, 6144, 0)], 449),     # k_conv1d_ip4, lines shorter than the block
    "pp_c2": ("1d", [(6000, 11999, 6144, 0)], 301),       # k_conv1d_pp 16x16x24 (HCONV_NO_IP=1), TMEM stash + accumulator
    "pp2_4096": ("1d", [(4000, 7999, 4096, 0)], 301),      # k_conv1d_pp2 (paired forward FFTs)
    "pp_small": ("1d", [(1024, 2047, 1024, 0)], 2001),      # k_conv1d_pp, several CTAs per SM
    "pp_centered": ("1d", [(1023, 1534, 512, 1)], 3),    # centered ping-pong
    "single_herm_tmem": ("1d", [(16383, 24574, 8192, 2)], 150),  # k_conv1d Hermitian, TMEM accumulator
    "single_stage_acc": ("1d", [(6000, 11999, 6144, 0)], 301),   # k_conv1d, accumulator staged by TMA (HCONV_NO_PP=1)
    "naive": ("1d", [(19, 37, 7, 0)], 4),                # direct-sum kernels
    "cols_2d": ("nd", [(256, 511, 256, 0), (192, 383, 128, 0)], 1),   # column tiles + inner conv
    "cols_3d_herm": ("nd", [(31, 46, 16, 1), (31, 46, 16, 1), (31, 46, 16, 2)], 1),
    "cols_3d_c5_like": ("nd", [(511, 766, 768, 1), (511, 766, 768, 1), (15, 22, 32, 2)], 1),  # c5 x/y tiles
    # one-buffer TMA column tiles (k_pfft_*_cols_tma1): blocks too long for two tile buffers, more tiles than CTAs
    "cols_2d_4096": ("nd", [(2048, 4095, 4096, 0), (320, 639, 128, 0)], 1),          # c4's x tiles: 2 columns of 4096 points
    "cols_2d_2048": ("nd", [(2047, 3070, 1024, 1), (1279, 1918, 1024, 2)], 1),        # centered, 3 residues, 4 columns of 2048 points
    "general_op": ("gen", [(1000, 1999, 1024, 0)], 3),   # conv1d_general (A = 3 product)
}


ENV = {"single_stage_acc": {"HCONV_NO_PP": "1"}, "pp_c2": {"HCONV_NO_IP": "1"}}
REPEAT = 3


def run(case):
    import os

    os.environ.update(ENV.get(case, {}))  # read once by the library at its first launch
    o = Oracle()
    kind, axes, C_ = CASES[case]
    rng = np.random.default_rng(7)
    shape = [((L + 1) // 2 if s == 2 else L) for (L, M, m, s) in axes]
    if kind in ("1d", "gen"):
        shape = [C_] + shape
    n_in = 3 if kind == "gen" else 2
    xs = [rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape) for _ in range(n_in)]
    if axes[-1][3] == 2:
        if kind == "nd":
            xs = [o.symmetrize([a[0] for a in axes], x) for x in xs]
        else:
            for x in xs:
                x[..., 0] = x[..., 0].real
    dev = [torch.from_numpy(x.copy()).cuda() for x in xs]
    if kind == "nd":
        plan = hconv.ConvPlanND([hconv.AxisSpec(L, M, m, hconv.Symmetry(s)) for L, M, m, s in axes])
        out = hconv.convolve_nd(dev[:2], plan.mult, plan, out=torch.empty_like(dev[0]))[0]
        ref = o.convolve(axes, xs[0], xs[1])
    elif kind == "gen":
        (L, M, m, s), = axes
        mult = hconv.builtin_mult_product(3)
        plan = hconv.Conv1dPlan(L, M, m, hconv.Symmetry(s), C_=C_, mult=mult)
        out = hconv.convolve(dev, mult, plan, out=torch.empty_like(dev[0]))[0]
        ref = o.convolve_general([axes[0]], xs, C_=C_)[0]
    else:
        (L, M, m, s), = axes
        plan = hconv.Conv1dPlan(L, M, m, hconv.Symmetry(s), C_=C_)
        out = hconv.convolve(dev[:2], plan.mult, plan, out=torch.empty_like(dev[0]))[0]
        ref = o.convolve([axes[0]], xs[0], xs[1], C_=C_)
    torch.cuda.synchronize()
    first = out.cpu().numpy()
    err = rel_l2(first, ref)
    assert np.isfinite(first).all(), "NaN / Inf in the output: a poisoned scratch value was read"
    for _ in range(REPEAT - 1):  # fresh output arrays, same inputs: bit-identical results
        if kind == "nd":
            again = hconv.convolve_nd(dev[:2], plan.mult, plan, out=torch.full_like(dev[0], float("nan")))[0]
        elif kind == "gen":
            again = hconv.convolve(dev, mult, plan, out=torch.full_like(dev[0], float("nan")))[0]
        else:
            again = hconv.convolve(dev[:2], plan.mult, plan, out=torch.full_like(dev[0], float("nan")))[0]
        torch.cuda.synchronize()
        assert np.array_equal(again.cpu().numpy(), first), "results differ between identical runs"
    print(f"{case}: kernel={plan.kernel(len(axes) - 1)} rel_l2={err:.2e} repeats={REPEAT} bit-identical")
    assert err <= 1e-12, err
    if DUMP:
        np.save(f"{DUMP}_{case}.npy", first)


DUMP = None

if __name__ == "__main__":
    args = sys.argv[1:]
    if args[:1] == ["--dump"]:
        DUMP, args = args[1], args[2:]
    names = args or list(CASES)
    for n in names:
        run(n)
