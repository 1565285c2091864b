"""Small invocations of every kernel family for compute-sanitizer (tools/sanitize.sh).

  python tools/sanitize_cases.py <case>      (one case per process: the sanitizer's report is
                                              per process)
Each case runs one convolution through the C ABI and checks it against the CPU oracle, so a run
that "passes" the sanitizer also computed the right numbers."""
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
    "pp_c2": ("1d", [(6000, 11999, 6144, 0)], 3),        # k_conv1d_pp 16x16x24, TMEM stash + accumulator
    "pp2_4096": ("1d", [(4000, 7999, 4096, 0)], 3),      # k_conv1d_pp2 (paired forward FFTs)
    "pp_small": ("1d", [(1024, 2047, 1024, 0)], 5),      # k_conv1d_pp, several CTAs per SM
    "pp_centered": ("1d", [(1023, 1534, 512, 1)], 3),    # centered ping-pong
    "single_herm_tmem": ("1d", [(16383, 24574, 8192, 2)], 2),  # k_conv1d Hermitian, TMEM accumulator
    "single_stage_acc": ("1d", [(6000, 11999, 6144, 0)], 3),   # k_conv1d, accumulator staged by TMA (HCONV_NO_PP=1)
    "naive": ("1d", [(19, 37, 7, 0)], 4),                # direct-sum kernels
    "cols_2d": ("nd", [(256, 511, 256, 0), (192, 383, 128, 0)], 1),   # column tiles + inner conv
    "cols_3d_herm": ("nd", [(31, 46, 16, 1), (31, 46, 16, 1), (31, 46, 16, 2)], 1),
    "general_op": ("gen", [(1000, 1999, 1024, 0)], 3),   # conv1d_general (A = 3 product)
}


ENV = {"single_stage_acc": {"HCONV_NO_PP": "1"}}


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
    err = rel_l2(out.cpu().numpy(), ref)
    print(f"{case}: kernel={plan.kernel(len(axes) - 1)} rel_l2={err:.2e}")
    assert err <= 1e-12, err


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        run(n)
