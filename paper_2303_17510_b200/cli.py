"""Command-line front end (SPEC.md:634-674 `verify | tune | bench`) over the B200 library.

  python -m paper_2303_17510_b200 verify [--kind complex|centered|hermitian] [--dims 1|2|3] [--max-L N] [--seed S]
  python -m paper_2303_17510_b200 tune   --L N (--M N | --ratio R) [--kind K] [--copies C] [--show-space]
  python -m paper_2303_17510_b200 bench  --L N|a..b (--M N | --ratio R) [--kind K] [--dims D] [--copies C] [--incremental]

verify checks the device path against brute-force direct sums computed here with numpy
(small sizes only), tune runs the device-timed planner and reports the choice
(`cached=true` when it came from the plan cache; the cache file is
$HCONV_PLAN_CACHE, default ~/.cache/hconv_b200_plans.csv), bench prints the SPEC's CSV rows
(mode,dims,L,M,strategy,median_ns,normalized_ns) for the hybrid (tuned), explicit-optimal and
explicit-next-power-of-two strategies, each configuration
spot-checked against the direct sum on small data before it is timed.
Exit status: 0 ok, 1 tolerance breach, 2 usage error.
"""
from __future__ import annotations

import argparse
import math
import os
import sys
from fractions import Fraction
from pathlib import Path

KINDS = {"complex": 0, "centered": 1, "hermitian": 2}
CSV_COLUMNS = "mode,dims,L,M,strategy,median_ns,normalized_ns"


def _usage(msg: str) -> None:
    print(f"usage error: {msg}", file=sys.stderr)
    raise SystemExit(2)


def _sizes(spec: str) -> list[int]:
    """`n` or `a..b` (inclusive)."""
    try:
        if ".." in spec:
            a, b = (int(x) for x in spec.split(".."))
            out = list(range(a, b + 1))
        else:
            out = [int(spec)]
    except ValueError:
        _usage(f"bad size list {spec!r}")
    if not out or min(out) < 1:
        _usage("empty or non-positive size list")
    return out


def _M(L: int, args) -> int:
    if args.M:
        return int(args.M)
    r = Fraction(args.ratio or "2")
    return max(L, math.ceil(r * L) - (1 if r == 2 and args.kind == "complex" else 0))


def _stored(L: int, kind: int) -> int:
    return (L + 1) // 2 if kind == 2 else L


# ------------------------------------------------------------------ direct sums --
def _box(kinds, Ls):
    """Per axis: logical lower bound lo and extent n of the full logical box, and the box position
    of stored index 0.  Complex: logical = stored; centered (and the outer axes of a Hermitian
    array): logical = stored - L//2; Hermitian (innermost): logical 0..K-1 stored, -(K-1)..K-1 full."""
    herm = kinds[-1] == 2
    lo, n, offs = [], [], []
    for k, (L, s) in enumerate(zip(Ls, kinds)):
        if s == 2:
            K = (L + 1) // 2
            lo.append(-(K - 1)), n.append(2 * K - 1), offs.append(K - 1)
        elif s == 1 or herm:
            lo.append(-(L // 2)), n.append(L), offs.append(0)
        else:
            lo.append(0), n.append(L), offs.append(0)
    return lo, n, offs


def _full(x, kinds, Ls):
    """The stored array embedded in its full logical box; Hermitian arrays get the points of
    negative innermost index from f(-x) = conj f(x) (0 where the mirror leaves the box)."""
    import numpy as np

    lo, n, offs = _box(kinds, Ls)
    F = np.zeros(n, complex)
    F[tuple(slice(o, o + m) for o, m in zip(offs, x.shape))] = x
    if kinds[-1] == 2:
        mir = [-2 * l - np.arange(m) for l, m in zip(lo, n)]
        ok = [(i >= 0) & (i < m) for i, m in zip(mir, n)]
        G = np.conj(F[np.ix_(*[np.clip(i, 0, m - 1) for i, m in zip(mir, n)])])
        mask = np.ones(n, bool)
        for k, v in enumerate(ok):
            shp = [1] * len(n)
            shp[k] = n[k]
            mask &= v.reshape(shp)
        G = np.where(mask, G, 0)
        K1 = offs[-1]  # box positions 0..K-2 hold the negative innermost indices
        F[..., :K1] = G[..., :K1]
    return F, lo, offs


def direct(x, y, kinds, Ls):
    """Linear convolution of the logical arrays on the stored output window (numpy FFTs of the
    whole logical boxes: exact up to rounding, an independent check of the padded algorithm)."""
    import numpy as np

    F, lo, offs = _full(x, kinds, Ls)
    G, _, _ = _full(y, kinds, Ls)
    shape = [2 * m - 1 for m in F.shape]
    H = np.fft.ifftn(np.fft.fftn(F, shape) * np.fft.fftn(G, shape))
    # box entry t of H has logical index 2 lo + t; stored output i has logical lo + offs + i
    return H[tuple(slice(o - l, o - l + m) for o, l, m in zip(offs, lo, x.shape))]


# ----------------------------------------------------------------------- verify --
def cmd_verify(args) -> int:
    import numpy as np
    import torch

    from . import hconv

    if args.max_L < 1:
        _usage("--max-L must be positive")
    kinds = [args.kind] if args.kind else list(KINDS)
    rng = np.random.default_rng(args.seed)
    worst = {}
    fails = 0
    for kname in kinds:
        kind = KINDS[kname]
        for L in range(1, args.max_L + 1):
            if kind == 2 and L % 2 == 0:
                continue  # Hermitian data: odd logical length 2K-1
            Ms = sorted({2 * L - 1 if L > 1 else 1, 2 * L}) if kind == 0 else [max(L, math.ceil(3 * L / 2))]
            for M in Ms:
                for m in sorted({1, max(1, L // 2), L, M}):
                    # per-axis kinds: a Hermitian array's outer axes are centered
                    kk = [kind if k == args.dims - 1 else (1 if kind == 2 else kind) for k in range(args.dims)]
                    shape = [_stored(L, s) for s in kk]
                    x = rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)
                    y = rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)
                    xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
                    if kind == 2:
                        for t in (xt, yt):
                            if args.dims > 1:
                                hconv.hermitian_symmetrize_boundary(t, [L] * args.dims)
                            else:
                                t[0] = t[0].real.to(t.dtype)
                        x, y = xt.cpu().numpy(), yt.cpu().numpy()
                    try:
                        if args.dims == 1:
                            plan = hconv.Conv1dPlan(L, M, m, hconv.Symmetry(kind), C_=1)
                            h = hconv.convolve([xt.view(1, -1), yt.view(1, -1)], plan.mult, plan,
                                               out=torch.empty_like(xt).view(1, -1))[0].view(-1)
                        else:
                            plan = hconv.ConvPlanND([hconv.AxisSpec(L, M, m, hconv.Symmetry(kind)) for _ in range(args.dims)])
                            h = hconv.convolve_nd([xt, yt], plan.mult, plan, out=torch.empty_like(xt))[0]
                    except NotImplementedError:
                        continue
                    ref = direct(x, y, kk, [L] * args.dims)
                    err = float(np.abs(h.cpu().numpy() - ref).max() / max(1e-300, np.abs(ref).max()))
                    key = (kname, args.dims)
                    worst[key] = max(worst.get(key, 0.0), err)
                    if not err <= 1e-11:
                        fails += 1
                        print(f"FAIL {kname} d={args.dims} L={L} M={M} m={m}: {err:.3e}")
    for (kname, d), e in sorted(worst.items()):
        print(f"{kname:9s} dims={d} max-L={args.max_L} worst relative error {e:.3e}")
    return 1 if fails else 0


# ------------------------------------------------------------------------- tune --
def _cache_default() -> None:
    if "HCONV_PLAN_CACHE" not in os.environ:
        p = Path.home() / ".cache" / "hconv_b200_plans.csv"
        p.parent.mkdir(parents=True, exist_ok=True)
        os.environ["HCONV_PLAN_CACHE"] = str(p)


def cmd_tune(args) -> int:
    _cache_default()
    from . import hconv

    kind = KINDS[args.kind]
    for L in _sizes(args.L):
        M = _M(L, args)
        params, rows, cached = hconv.tune_1d(L, M, hconv.Symmetry(kind), C_=args.copies)
        print(f"L={L} M={M} kind={args.kind} copies={args.copies}: m={params.m} p={params.p} q={params.q} "
              f"n={params.n} block={params.blockLength()} cached={'true' if cached else 'false'}")
        if args.show_space:
            for r in rows:
                print(f"  m={r['m']:6d} p={r['p']:4d} q={r['q']:5d} n={r['n']:4d} block={r['block']:6d} "
                      f"median_ms={r['median_ms']:.4f}" + (" explicit" if r.get('explicit') else ""))
    return 0


# ------------------------------------------------------------------------ bench --
def _time(run, reps: int = 7) -> float:
    import torch

    run()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e6)
    ts.sort()
    return ts[len(ts) // 2]


def cmd_bench(args) -> int:
    import numpy as np
    import torch

    from . import hconv

    _cache_default()
    kind = KINDS[args.kind]
    d = args.dims
    if args.csv_header == "on":
        print(CSV_COLUMNS)
    for L in _sizes(args.L):
        M = _M(L, args)
        S = _stored(L, kind)
        # explicit-optimal: the smallest explicit size >= M with a radix kernel (q = 1);
        # explicit-pow2: the next power of two >= M
        strategies = [("hybrid", None), ("explicit-pow2", 1 << (M - 1).bit_length())]
        opt = next((m for m in range(M, 4 * M + 1) if _has_kernel(hconv, L, M, m, kind)), None)
        if opt is not None:
            strategies.insert(1, ("explicit-optimal", opt))
        for name, m in strategies:
            try:
                if d == 1:
                    plan = hconv.Conv1dPlan(L, M, m, hconv.Symmetry(kind), C_=args.copies)
                    shape = (args.copies, S)
                    run_fn = hconv.convolve
                else:
                    syms = [hconv.Symmetry(1 if kind == 2 else kind)] * (d - 1) + [hconv.Symmetry(kind)]
                    plan = hconv.ConvPlanND([hconv.AxisSpec(L, M, m, s) for s in syms])
                    shape = plan.shape()
                    run_fn = hconv.convolve_nd
                f = torch.empty(shape, dtype=torch.complex128, device="cuda")
                g = torch.empty_like(f)
                hconv.fill_uniform(f, args.seed, 0)
                hconv.fill_uniform(g, args.seed, 1)
                out = torch.empty_like(f)
                if not _spot_check(hconv, L, M, plan, kind, d):
                    print(f"# {name} L={L} M={M}: spot check failed", file=sys.stderr)
                    return 1
                ns = _time(lambda: run_fn([f, g], plan.mult, plan, out=out))
            except (NotImplementedError, ValueError) as e:
                print(f"# {name} L={L} M={M}: {e}", file=sys.stderr)
                continue
            N = L ** d
            norm = ns / (N * math.log2(max(N, 2)))
            print(f"{args.kind},{d},{L},{M},{name},{ns:.0f},{norm:.6g}", flush=True)
    return 0


def _has_kernel(hconv, L, M, m, kind) -> bool:
    """m is an explicit size (q = 1: one residue block covers the whole padded length) with a
    radix kernel (direct sums only for blocks of at most 64 points)."""
    try:
        p = hconv.deriveParams(L, M, m, hconv.Symmetry(kind))
    except ValueError:
        return False
    if p.q != 1:
        return False
    try:
        plan = hconv.Conv1dPlan(L, M, m, hconv.Symmetry(kind), C_=1)
        return plan.kernel() != "direct" or p.blockLength() <= 64
    except (NotImplementedError, ValueError):
        return False


def _spot_check(hconv, L, M, plan, kind, d) -> bool:
    """every benchmarked configuration is verified once on small random data (the
    same plan parameters, a few copies / one small array) against the direct sum."""
    import numpy as np
    import torch

    if L ** d > 4096:
        return True  # direct sums above this size are too slow for a spot check
    rng = np.random.default_rng(0)
    S = _stored(L, kind)
    shape = (S,) if d == 1 else plan.shape()
    x = rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)
    y = rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)
    xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    if kind == 2:
        if d == 1:
            xt[0] = xt[0].real.to(xt.dtype)
            yt[0] = yt[0].real.to(yt.dtype)
        else:
            hconv.hermitian_symmetrize_boundary(xt, [L] * d)
            hconv.hermitian_symmetrize_boundary(yt, [L] * d)
        x, y = xt.cpu().numpy(), yt.cpu().numpy()
    kk = [kind] if d == 1 else [1 if kind == 2 else kind] * (d - 1) + [kind]
    if d == 1:
        p1 = hconv.Conv1dPlan(L, M, plan.params.m, hconv.Symmetry(kind), C_=1)
        h = hconv.convolve([xt.view(1, -1), yt.view(1, -1)], p1.mult, p1, out=torch.empty_like(xt).view(1, -1))[0].view(-1)
    else:
        h = hconv.convolve_nd([xt, yt], plan.mult, plan, out=torch.empty_like(xt))[0]
    ref = direct(x, y, kk, [L] * d)
    return float(np.abs(h.cpu().numpy() - ref).max() / max(1e-300, np.abs(ref).max())) <= 1e-11


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2303_17510_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)

    def shared(p, need_sizes):
        p.add_argument("--kind", choices=sorted(KINDS), default="complex")
        p.add_argument("--dims", type=int, choices=(1, 2, 3), default=1)
        if need_sizes:
            p.add_argument("--L", required=True, help="n or a..b")
            p.add_argument("--M", default=None)
            p.add_argument("--ratio", default=None, help="M/L as a decimal or fraction (default 2: M = 2L-1 complex)")
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--csv-header", choices=("on", "off"), default="on")
        p.add_argument("--threads", type=int, default=1, help="reserved (the device path is one GPU)")

    v = sub.add_parser("verify", help="device path vs direct sums over a size sweep")
    shared(v, False)
    v.set_defaults(kind=None)
    v.add_argument("--max-L", type=int, default=24)
    t = sub.add_parser("tune", help="device-timed planner choice (cached)")
    shared(t, True)
    t.add_argument("--copies", type=int, default=1024)
    t.add_argument("--show-space", action="store_true")
    b = sub.add_parser("bench", help="CSV timings of hybrid vs explicit strategies")
    shared(b, True)
    b.add_argument("--copies", type=int, default=1024)
    b.add_argument("--incremental", action="store_true", help="sweep every L of the range (default for a..b)")
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    if args.threads != 1:
        _usage("--threads is reserved and must be 1")
    if args.cmd == "verify":
        return cmd_verify(args)
    if args.cmd == "tune":
        return cmd_tune(args)
    return cmd_bench(args)


if __name__ == "__main__":
    raise SystemExit(main())
