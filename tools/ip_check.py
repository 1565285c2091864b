"""In-place kernel check: one 1D complex convolution against an explicit torch.fft route (all rows)
and the CPU oracle (first rows), with CUDA-event timing.  Usage: ip_check.py L M m C"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2303_17510_b200 import hconv  # noqa: E402

L, M, m, C_ = (int(x) for x in sys.argv[1:5])
plan = hconv.Conv1dPlan(L, M, m, hconv.Symmetry.Complex, C_=C_)
f = torch.empty((C_, L), dtype=torch.complex128, device="cuda")
g = torch.empty_like(f)
hconv.fill_uniform(f, 1, 0)
hconv.fill_uniform(g, 1, 1)
out = torch.empty_like(f)
hconv.convolve([f, g], plan.mult, plan, out=out)
torch.cuda.synchronize()
n = 1
while n < 2 * L:
    n *= 2
ref = torch.fft.ifft(torch.fft.fft(f, n=n, dim=1) * torch.fft.fft(g, n=n, dim=1), dim=1)[:, :L]
err = (out - ref).abs().max().item() / ref.abs().max().item()
print(f"max rel err vs torch.fft (all {C_} rows): {err:.3e}")
try:
    from oracle_lib import Oracle, rel_l2
    o = Oracle()
    k = min(C_, 8)
    r = o.convolve([(L, M, plan.params.m, 0)], f[:k].cpu().numpy(), g[:k].cpu().numpy(), C_=k)
    print(f"rel_l2 vs oracle ({k} rows): {rel_l2(out[:k].cpu().numpy(), r):.3e}")
except Exception as e:  # noqa: BLE001
    print("oracle check skipped:", e)
outs = [out.clone()]
for _ in range(2):
    hconv.convolve([f, g], plan.mult, plan, out=out)
    outs.append(out.clone())
print("bit-identical runs:", all(torch.equal(outs[0], x) for x in outs[1:]))
ts = []
for _ in range(25):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hconv.convolve([f, g], plan.mult, plan, out=out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
p = plan.params
print(f"L={L} M={M} m={p.m} p={p.p} q={p.q} n={p.n} C={C_} kernel={plan.kernel()} ms={ts[12]:.4f} min={ts[0]:.4f}")
