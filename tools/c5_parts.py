"""c5 decomposition parts on one GPU (diagnostics): the z-line subconvolutions as a 1D Hermitian
batch (768 x 768 lines of L = 511, M = 766) for every z block size with a kernel, and whole c5
convolutions for fixed per-axis m.  CUDA events, median of 5 after warm-up."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2303_17510_b200 import hconv  # noqa: E402


def timed(fn, reps=5):
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


L, M = 511, 766
lines = int(sys.argv[1]) if len(sys.argv) > 1 else 768 * 768
f = torch.empty((lines, 256), dtype=torch.complex128, device="cuda")
g = torch.empty_like(f)
hconv.fill_uniform(f, 1, 0)
hconv.fill_uniform(g, 1, 1)
f[:, 0] = f[:, 0].real.to(f.dtype)
g[:, 0] = g[:, 0].real.to(g.dtype)
o = torch.empty_like(f)
for m in (256, 384, 512, 768, 1024):
    try:
        plan = hconv.Conv1dPlan(L, M, m, hconv.Symmetry.Hermitian, C_=lines)
    except (NotImplementedError, ValueError) as e:
        print(f"z m={m}: {e}")
        continue
    p = plan.params
    t = timed(lambda: hconv.convolve([f, g], plan.mult, plan, out=o))
    print(f"z-lines m={m} p={p.p} q={p.q} n={p.n} block={p.blockLength()} kernel={plan.kernel()} {t:.3f} ms")
del f, g, o
torch.cuda.empty_cache()
shape = (511, 511, 256)
f = torch.empty(shape, dtype=torch.complex128, device="cuda")
g = torch.empty_like(f)
hconv.fill_uniform(f, 1, 0)
hconv.fill_uniform(g, 1, 1)
hconv.hermitian_symmetrize_boundary(f, (L, L, L))
hconv.hermitian_symmetrize_boundary(g, (L, L, L))
o = torch.empty_like(f)
for ms in [(768, 768, 1024), (768, 768, 768), (768, 768, 512), (768, 768, 256), (256, 768, 768), (512, 512, 768)]:
    try:
        plan = hconv.ConvPlanND([hconv.AxisSpec(L, M, ms[0], hconv.Symmetry.Centered),
                                 hconv.AxisSpec(L, M, ms[1], hconv.Symmetry.Centered),
                                 hconv.AxisSpec(L, M, ms[2], hconv.Symmetry.Hermitian)])
    except (NotImplementedError, ValueError) as e:
        print(f"c5 m={ms}: {e}")
        continue
    t = timed(lambda: hconv.convolve_nd([f, g], plan.mult, plan, out=o), reps=3)
    print(f"c5 m={ms} n={[p.n for p in plan.params]} {t:.3f} ms")
