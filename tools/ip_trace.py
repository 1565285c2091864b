"""Phase trace of the in-place kernel (HCONV_TRACE=1): per-phase clock deltas of three warps."""
import os, subprocess, sys, re
env = dict(os.environ, HCONV_TRACE="1")
r = subprocess.run([sys.executable, "tools/ab_conv.py", "6000", "11999", "6144", "4096"], env=env, capture_output=True, text=True)
lines = [l for l in r.stderr.splitlines() if "ip trace" in l]
# the last launch's three lines
names = ["start", "wait_f", "P0f", "wait_g", "P0g", "waitX", "P1f", "waitY", "P1g", "waitGF", "ldF+waitGG", "P2", "tma_f", "waitGI", "I1", "waitY", "I0"]
import os
PER = int(os.environ.get("PER", "17"))
for l in lines[-3:]:
    v = [int(x) for x in l.split("]")[1].split()]
    print(l.split("]")[0] + "]", "stamps", len(v))
    per = PER if 'slot 2' not in l else PER - (1 if PER == 17 and os.environ.get('W11_SHORT') else 0)
    nres = len(v) // per
    import collections
    acc = collections.defaultdict(list)
    for k in range(1, nres):  # skip the first residue
        seg = v[k * per:(k + 1) * per]
        prev_end = v[k * per - 1]
        acc["gap"].append(seg[0] - prev_end)
        for i in range(1, per):
            acc[f"{i:02d}_{names[i]}"].append(seg[i] - seg[i - 1])
    tot = 0
    for key in sorted(acc):
        m = sum(acc[key]) / len(acc[key])
        tot += m
        print(f"   {key:12s} mean {m:8.0f}  min {min(acc[key]):6d} max {max(acc[key]):6d}")
    print(f"   total per residue {tot:.0f}")
print(r.stdout[-300:])
