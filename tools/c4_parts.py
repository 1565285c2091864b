"""c4 decomposition parts on one GPU (diagnostics): whole 2048 x 2048 (M = 4095) complex convolutions
for fixed per-axis m, and the outer x passes alone (hconv_pfft_*_lines is not needed: the plan with
an inner direct product is not available, so the difference to the inner batch is reported).
CUDA events, median of 7 after warm-up."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2303_17510_b200 import hconv  # noqa: E402


def timed(fn, reps=7):
    fn()
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


L, M = 2048, 4095
quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
for m, lines in (((4096, 4096),) if quick else ((4096, 4096), (2048, 2048), (2048, 4096))):
    f = torch.empty((lines, L), dtype=torch.complex128, device="cuda")
    g = torch.empty_like(f)
    hconv.fill_uniform(f, 1, 0)
    hconv.fill_uniform(g, 1, 1)
    o = torch.empty_like(f)
    try:
        plan = hconv.Conv1dPlan(L, M, m, hconv.Symmetry.Complex, C_=lines)
    except (NotImplementedError, ValueError) as e:
        print(f"inner m={m}: {e}")
        continue
    t = timed(lambda: hconv.convolve([f, g], plan.mult, plan, out=o))
    p = plan.params
    print(f"inner lines={lines} m={m} n={p.n} kernel={plan.kernel()} {t:.3f} ms")
    del f, g, o
shape = (L, L)
f = torch.empty(shape, dtype=torch.complex128, device="cuda")
g = torch.empty_like(f)
hconv.fill_uniform(f, 1, 0)
hconv.fill_uniform(g, 1, 1)
o = torch.empty_like(f)
for ms in ([(4096, 4096)] if quick else [(4096, 4096), (2048, 4096), (1024, 4096), (4096, 2048), (2048, 2048), (1024, 2048)]):
    try:
        plan = hconv.ConvPlanND([hconv.AxisSpec(L, M, ms[0], hconv.Symmetry.Complex),
                                 hconv.AxisSpec(L, M, ms[1], hconv.Symmetry.Complex)])
    except (NotImplementedError, ValueError) as e:
        print(f"c4 m={ms}: {e}")
        continue
    t = timed(lambda: hconv.convolve_nd([f, g], plan.mult, plan, out=o))
    print(f"c4 m={ms} n={[p.n for p in plan.params]} {t:.3f} ms")
