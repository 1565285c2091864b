"""A/B timing of one 1D convolution configuration (CUDA events, median of 20 after warm-up);
prints ms per convolution and a checksum to compare variants (env knobs set by the caller)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2303_17510_b200 import hconv  # noqa: E402

L, M, m, C_ = (int(x) for x in sys.argv[1:5])
sym = int(sys.argv[5]) if len(sys.argv) > 5 else 0
plan = hconv.Conv1dPlan(L, M, m, hconv.Symmetry(sym), C_=C_)
S = plan.params.dataLength()
f = torch.empty((C_, S), dtype=torch.complex128, device="cuda")
g = torch.empty_like(f)
hconv.fill_uniform(f, 1, 0)
hconv.fill_uniform(g, 1, 1)
out = torch.empty_like(f)
for _ in range(3):
    hconv.convolve([f, g], plan.mult, plan, out=out)
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hconv.convolve([f, g], plan.mult, plan, out=out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
torch.save(out[:64].cpu(), f"/tmp/ab_{L}_{m}.pt") if len(sys.argv) > 6 else None
print(f"L={L} M={M} m={m} C={C_} kernel={plan.kernel()} ms={ts[10]:.4f} sum={out.abs().sum().item():.12e}")
