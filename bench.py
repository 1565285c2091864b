#!/usr/bin/env python3
"""Benchmark of the hybrid-dealiased convolution path on B200 (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference] [--config c1..c5]

Workload per GPU count (BASELINE.json: 1 GPU for every config, 2/4/8 GPUs for the partitioned
2D/3D configs):
  N = 1  configs[1] (c2: 1D complex, L = 6000, M = 11999, batch 4096, planner-chosen m/p/q) as
         the headline line; the other four configurations ride along in "configs".
  N > 1  configs[4] (c5: 3D Hermitian 511^2 x 256, M = 766) slab-decomposed over the N GPUs
         (strong scaling, NCCL exchanges inside the library); T_1 (the same problem on one GPU,
         measured in the same run on rank 0) and c2 sharded over the ranks ride along.
  --gpus N without torchrun: bench.py re-launches itself under torch.distributed.run.
A step is one convolution of the whole workload.  Inputs are resident in HBM for `value`;
`e2e` copies them from pinned host memory and the result back inside every timed step.

--impl reference times the reference's CPU path on the host cores: the reference's own code
cannot be built (FFTW++/FFTW absent), so this is the CPU restatement in oracle/
(kind "port"), rank 0 only, on a bounded sample per step (1D: copies of the batch; N-D: one
whole convolution).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

A, B = 2, 1
L2_BYTES = 126 * 1024 * 1024
CONFIGS = {
    # name: (dims, [(L, M, symmetry)], batch C)
    "c1": (1, [(1024, 2047, 0)], 1024),
    "c2": (1, [(6000, 11999, 0)], 4096),
    "c3": (1, [(16383, 24574, 2)], 2048),
    "c4": (2, [(2048, 4095, 0), (2048, 4095, 0)], 1),
    "c5": (3, [(511, 766, 1), (511, 766, 1), (511, 766, 2)], 1),
}
WORKLOAD = {
    "c1": "1D complex binary convolution L=1024 M=2047 batch 1024",
    "c2": "1D complex binary convolution L=6000 M=11999 batch 4096 (planner-chosen m/p/q)",
    "c3": "1D centered Hermitian binary convolution K=8192 (L=16383) M=24574 batch 2048",
    "c4": "2D complex binary convolution 2048x2048 M=4095",
    "c5": "3D centered Hermitian binary convolution 511x511x256(stored) M=766",
}


def stored(L, sym):
    return (L + 1) // 2 if sym == 2 else L


def config_sizes(name):
    dims, axes, C_ = CONFIGS[name]
    shape = [stored(L, s) for (L, M, s) in axes]
    n_out = C_ * math.prod(shape)
    return dims, axes, C_, shape, n_out


def working_set(name):
    """bytes of one set of inputs and outputs (A + B arrays)."""
    return 16 * (A + B) * config_sizes(name)[4]


def input_sets(name, world=1):
    """input sets rotated between timed steps so that consecutive steps never find their data
    in L2: >= 2 x L2 in total; 1 when one set is already larger."""
    ws = working_set(name) // (world if CONFIGS[name][0] > 1 else 1)
    return 1 if ws >= 2 * L2_BYTES else math.ceil(2 * L2_BYTES / ws)


def config_dict(name, world=1):
    """the workload identity, identical in both arms' lines (no implementation details)."""
    dims, axes, C_, shape, n_out = config_sizes(name)
    sets = input_sets(name, world)
    l2 = (f"{sets} input sets rotated between steps (>= 2 x 126 MB L2 in total)" if sets > 1
          else f"inputs + outputs ({working_set(name) / 1e6:.0f} MB) larger than the 126 MB L2")
    batch = C_ * (world if dims == 1 else 1)
    return {"workload": WORKLOAD[name], "config": name, "global_batch": batch, "l2": l2}


def algorithmic(name):
    """bytes / flops per step: 16 (A N_in + B N_out), 5 N log2 N per complex
    padded-axis FFT (2.5 for the Hermitian axis) at N = M, mult 6 (complex) / 1 (real) flops."""
    dims, axes, C_, shape, n_out = config_sizes(name)
    nbytes = 16 * (A * n_out + B * n_out)
    if dims == 1:
        L, M, s = axes[0]
        fft = (2.5 if s == 2 else 5.0) * M * math.log2(M)
        flops = C_ * ((A + B) * fft + (1 if s == 2 else 6) * M)
    elif dims == 2:
        (L, M, _), _ = axes
        flops = (A + B) * (L * 5 * M * math.log2(M) + M * 5 * M * math.log2(M)) + 6 * M * M
    else:
        L, M, _ = axes[0]
        K = shape[2]
        flops = (A + B) * (L * K * 5 * M * math.log2(M) + M * K * 5 * M * math.log2(M) + M * M * 2.5 * M * math.log2(M)) + M ** 3
    return nbytes, flops


def peaks():
    """roofline denominators: measured HBM copy (MEASURED_PEAKS.json) and measured FP64 DFMA
    throughput (profiles/r01_step0_fp64.json; MEASURED_PEAKS.json has no FP64 figure)."""
    hbm, src_h = 6453.4, "MEASURED_PEAKS.json (fallback value)"
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        hbm, src_h = float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    fp64, src_f = 34.16, "measured DFMA (profiles/r01_step0_fp64.json)"
    q = REPO / "profiles" / "r01_step0_fp64.json"
    if q.exists():
        vals = [json.loads(l)["tflops"] for l in q.read_text().splitlines() if '"dfma"' in l]
        if vals:
            fp64 = max(vals)
    return hbm, src_h, fp64, src_f


def ncu_traffic(name):
    """DRAM bytes per launch of the dominant kernel from the newest ncu capture in profiles/."""
    for r in ("r02", "r01"):
        tp = REPO / "profiles" / f"{r}_{name}_ncu_traffic.json"
        if tp.exists():
            return json.loads(tp.read_text()).get("dram_bytes_per_launch")
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-i",
                                       str(self.gpu), "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        # nvidia-smi's first start on a fresh box can take seconds (NVML init): wait for its first
        # sample so that its start-up does not fall inside the timed region
        t0 = time.time()
        while self.p and time.time() - t0 < 10.0:
            self.f.flush()
            if Path(self.f.name).stat().st_size > 0:
                break
            time.sleep(0.05)
        time.sleep(0.2)
        return self

    def __exit__(self, *exc):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        rows = [l.split(", ") for l in Path(self.f.name).read_text().splitlines() if l.strip()]
        clocks, reasons, maxes = [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                clocks.append(float(r[1]))
                maxes.append(float(r[2]))
                for n, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                pass
        load = [c for c in clocks if c > 500] or clocks
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(clocks)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def default_config(args):
    return args.config or ("c2" if args.gpus <= 1 else "c5")


# ------------------------------------------------------------------ CPU arm ------
# candidate subtransform sizes of the CPU baseline's own tuning probe (hybrid, explicit, pow2)
CPU_CANDIDATES = {"c1": [256, 512, 1024, 2048], "c2": [1024, 1536, 2000, 2048, 3000, 3072, 4096, 6000, 6144, 12000],
                  "c3": [2048, 4096, 8192, 12288]}
# N-D: the explicit candidate per axis (the oracle's m = 0 default) and the paper's hybrid sizes
CPU_ND_M = {"c4": [4096, 4096], "c5": [256, 256, 256]}


class CpuArm:
    """Oracle (CPU restatement, TEST INFRASTRUCTURE) on a bounded sample of the workload: 1D, a
    probe sizes the sample and each call convolves `rows` copies of the batch; N-D, each call is
    one whole convolution (the problem does not split into independent copies)."""

    def __init__(self, name, m=None, threads=None):
        sys.path.insert(0, str(REPO / "tests"))
        from oracle_lib import Oracle

        self.o = Oracle()
        self.name = name
        self.threads = threads or os.cpu_count()
        self.o.lib.oracle_set_threads(self.threads)
        self.dims, self.axes, self.C, self.shape, n_out = config_sizes(name)
        if self.dims > 1:
            self.m = list(m) if m else CPU_ND_M[name]
            self.rows = 1
            return
        self.L, self.M, self.s = self.axes[0]
        self.S = self.shape[0]
        probe = max(self.threads, 8)
        self.rows = probe
        if m:
            self.m = m[0] if isinstance(m, (list, tuple)) else m
            self.per_row = self.run()[1] / probe
        else:
            # the CPU path's own hybrid choice: time a probe of each candidate m (the paper's tuner,
            # PAPER.md:894-914, on the host cores) and keep the fastest
            best = None
            for mc in CPU_CANDIDATES[name]:
                self.m = mc
                dt = self.run()[1]
                if best is None or dt < best[1]:
                    best = (mc, dt)
            self.m = best[0]
            self.per_row = best[1] / probe

    def size_for(self, seconds):
        if self.dims == 1:
            self.rows = int(min(self.C, max(self.threads, seconds / max(self.per_row, 1e-9))))

    def run(self):
        if self.dims > 1:
            import numpy as np

            n = math.prod(self.shape)
            f = self.o.uniform(1, 0, n).reshape(self.shape)
            g = self.o.uniform(1, 1, n).reshape(self.shape)
            if self.dims == 3:
                Ls = [L for (L, M, s) in self.axes]
                f, g = self.o.symmetrize(Ls, f), self.o.symmetrize(Ls, g)
            ax = [(L, M, mk, s) for (L, M, s), mk in zip(self.axes, self.m)]
            t0 = time.perf_counter()
            self.o.convolve(ax, f, g)
            dt = time.perf_counter() - t0
            return n / dt, dt
        f = self.o.uniform(1, 0, self.rows * self.S).reshape(self.rows, self.S)
        g = self.o.uniform(1, 1, self.rows * self.S).reshape(self.rows, self.S)
        t0 = time.perf_counter()
        self.o.convolve([(self.L, self.M, self.m, self.s)], f, g, C_=self.rows)
        dt = time.perf_counter() - t0
        return self.rows * self.S / dt, dt

    def sample(self, dt):
        if self.dims > 1:
            return f"one whole convolution per step (m={self.m}), {dt:.2f} s"
        return f"{self.rows} of {self.C} copies per step (m={self.m}), {dt:.2f} s per step"


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    name = default_config(args)
    dims, axes, C_, shape, n_out = config_sizes(name)
    ms = [int(x) for x in str(args.m).split(",")] if args.m else None
    arm = CpuArm(name, ms)
    steps, warmup = args.steps, args.warmup
    if dims > 1:  # one whole N-D convolution is the bounded sample; time it once
        steps, warmup = 1, 0
    arm.size_for(max(0.5, 120.0 / (steps + warmup)))  # whole run ~2 minutes
    vals, dts = [], []
    for i in range(warmup + steps):
        v, dt = arm.run()
        if i >= warmup:
            vals.append(v)
            dts.append(dt)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "complex128 dealiased-convolution output points/s", "value": value,
        "unit": "points/s", "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
        "ms_per_step": n_out / value * 1e3 if dims == 1 else statistics.median(dts) * 1e3,
        "higher_is_better": True, "scaling": "weak" if dims == 1 else "strong", "vs_baseline": None,
        "dtype": "complex128 (f64)", "data": "synthetic (counter-based uniform[-1,1], seed 1)",
        "config": config_dict(name, args.gpus),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": arm.threads, "kind": "port",
                         "sample": arm.sample(statistics.median(dts)) +
                         "; CPU restatement (oracle/), the reference's FFTW++/FFTW path is not buildable here"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm ------
def launches_per_step(params):
    """kernels one convolution launches: 1D = 1 fused conv; N-D = per outer residue A forward +
    inner + B backward."""
    if len(params) == 1:
        return 1
    return params[0].n * (A + launches_per_step(params[1:]) + B)


class Dist:
    def __init__(self, rank, world, local):
        self.rank, self.world, self.local = rank, world, local

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier(device_ids=[self.local])

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], device=f"cuda:{self.local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())


def _timed(step, steps, stream, dd: Dist, sampler=None):
    """device time of `steps` calls of step(i) (CUDA events on the launching stream, barrier +
    synchronize on both sides, max over ranks), in ms."""
    import torch

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dd.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    dd.barrier()
    return dd.max(e0.elapsed_time(e1))


def measure(name, args, dd: Dist, headline: bool):
    """One configuration: plan (planner outside the timed region), W warm-up steps, K timed steps
    with rotating input sets, the end-to-end host-buffer steps; returns the line's fields."""
    import torch

    from paper_2303_17510_b200 import hconv

    dev = torch.device("cuda", dd.local)
    stream = torch.cuda.current_stream()
    dims, axes, C_, shape, n_out = config_sizes(name)
    slab = dims > 1 and (dd.world > 1 or args.slab)
    steps, warmup = (args.steps, args.warmup) if headline else (min(args.steps, 10), 3)
    ms = [None] * dims
    if args.m and headline:
        vals = [int(x) for x in str(args.m).split(",")]
        ms = vals if len(vals) == dims else [vals[0]] * dims
    sc = None
    if dims == 1:
        L, M, s = axes[0]
        plan = hconv.Conv1dPlan(L, M, ms[0], hconv.Symmetry(s), C_=C_, device=dd.local)
        params = [plan.params]
        kernel = plan.kernel()
    elif slab:
        from paper_2303_17510_b200.distributed import SlabAxis, SlabConvND, choose_sizes

        if None in ms:
            ms = choose_sizes(axes, device=dev)
        sc = SlabConvND([SlabAxis(L, M, mk, s) for (L, M, s), mk in zip(axes, ms)], chunks=args.chunks, device=dev)
        params = [sc.params(k) for k in range(dims)]
        plan = None
        kernel = "slab"
    else:
        plan = hconv.ConvPlanND([hconv.AxisSpec(L, M, mk, hconv.Symmetry(s)) for (L, M, s), mk in zip(axes, ms)],
                                device=dd.local)
        params = plan.params
        kernel = plan.kernel(len(params) - 1)
    sets = input_sets(name, dd.world) if not slab else 1
    full_shape = (C_, *shape) if dims == 1 else tuple(shape)
    ins, outs = [], []
    for k in range(sets):
        f = torch.empty(full_shape, dtype=torch.complex128, device=dev)
        g = torch.empty_like(f)
        first = dd.rank * f.numel() if dims == 1 else 0  # 1D: each rank owns its own slice of the global batch
        hconv.fill_uniform(f, 1 + k, 0, first)
        hconv.fill_uniform(g, 1 + k, 1, first)
        if dims == 3:
            hconv.hermitian_symmetrize_boundary(f, [L for (L, M, s) in axes])
            hconv.hermitian_symmetrize_boundary(g, [L for (L, M, s) in axes])
        if slab:
            f, g = f[sc.x0:sc.x0 + sc.nx].clone(), g[sc.x0:sc.x0 + sc.nx].clone()  # this rank's x-slabs
            torch.cuda.empty_cache()
        ins.append((f, g))
        outs.append(torch.empty_like(f))

    if slab:
        def step(i):
            sc.convolve(list(ins[0]), out=[outs[0]])
    elif args.no_graph:
        run = hconv.convolve if dims == 1 else hconv.convolve_nd

        def step(i):
            f, g = ins[i % sets]
            run([f, g], plan.mult, plan, out=outs[i % sets])
    else:
        # the step's kernels captured once per input set in a CUDA graph (warm-up and capture
        # outside the timed region); each timed step replays one whole convolution
        caps = [hconv.CapturedConvolution([f, g], plan.mult, plan, out=o) for (f, g), o in zip(ins, outs)]

        def step(i):
            caps[i % sets]()
    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    sampler = ClockSampler(dd.local) if headline else None
    if sampler:
        sampler.__enter__()
    try:
        t_ms = _timed(step, steps, stream, dd)
    finally:
        if sampler:
            sampler.__exit__()
    ms_step = t_ms / steps
    value = (1 if dims > 1 else dd.world) * n_out * steps / (t_ms * 1e-3)

    # e2e through the public host-buffer API (hconv.convolve_host, the reference's calling
    # convention): every step copies both inputs from pinned host memory to the device and the
    # result back (1D: in chunks, copies and compute overlapped on three streams)
    f, g = ins[0]
    hf = f.cpu().pin_memory()
    hg = g.cpu().pin_memory()
    ho = torch.empty_like(hf).pin_memory()

    def step_host(i):
        if slab:  # host slabs in, device slab convolution, host slab out
            fd, gd = hf.to(dev, non_blocking=True), hg.to(dev, non_blocking=True)
            ho.copy_(sc.convolve([fd, gd])[0], non_blocking=True)
            torch.cuda.current_stream().synchronize()
        else:
            hconv.convolve_host([hf, hg], plan.mult, plan, out=ho)

    for i in range(2):
        step_host(i)
    e2e_steps = max(1, min(steps, 5))
    # the host call is synchronous: events on the (idle) current stream bracket whole calls
    e2e_ms = _timed(step_host, e2e_steps, stream, dd)
    e2e_value = (1 if dims > 1 else dd.world) * n_out * e2e_steps / (e2e_ms * 1e-3)

    hbm, src_h, fp64, src_f = peaks()
    nbytes, flops = algorithmic(name)
    per_gpu = dd.world if dims > 1 else 1  # the roofline is per GPU: N-D shares one problem
    nbytes, flops = nbytes / per_gpu, flops / per_gpu
    t_s = ms_step * 1e-3
    achieved_tf = flops / t_s / 1e12
    t_roof = max(nbytes / (hbm * 1e9), flops / (fp64 * 1e12))
    launches = steps * launches_per_step(params)
    if slab:  # per y residue: A forward, the inner launches per k-chunk, B backward (copies not counted)
        inner = launches_per_step([params[0]] + list(params[2:]))
        launches = steps * params[1].n * (A + slab_chunks(_block(params[1]), dd.world, args.chunks) * inner + B)
    out = {
        "value": value, "ms_per_step": ms_step, "steps": steps, "warmup": warmup,
        "plan": [dict(m=p.m, p=p.p, q=p.q, n=p.n, block=_block(p), regime=_regime(p)) for p in params],
        "kernel": kernel,
        "launch": "direct API calls" if (slab or args.no_graph) else "CUDA graph replay of the API call (captured once per input set)",
        "input_sets": sets,
        "roofline": {
            "bound": "fp64", "achieved": achieved_tf, "peak": fp64, "unit": "TFLOP/s", "frac": achieved_tf / fp64,
            "traffic": ncu_traffic(name) if not slab else None, "peak_source": src_f,
            "hbm": {"achieved": nbytes / t_s / 1e9, "peak": hbm, "unit": "GB/s", "frac": nbytes / t_s / 1e9 / hbm,
                    "peak_source": src_h},
            "north_star_frac": t_roof / t_s,
            "algorithmic": {"bytes": nbytes, "flops": flops, "per": "GPU" if per_gpu > 1 else "step"},
        },
        "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": 2 * f.numel() * 16,
                "d2h_bytes_per_step": f.numel() * 16, "steps": e2e_steps},
        "gpu_launches": launches,
    }
    if sampler:
        out["clocks"] = sampler.summary()
    if slab:
        By = _block(params[1])
        xch = (A + B) * shape[0] * By * (shape[2] if dims == 3 else 1) * 16 * params[1].n
        per_gpu_bytes = xch * (dd.world - 1) / dd.world ** 2
        out["exchange"] = {"bytes_per_gpu_per_step": per_gpu_bytes, "chunks": slab_chunks(By, dd.world, args.chunks),
                           "lower_bound_gbs": per_gpu_bytes / t_s / 1e9,
                           "how": "NCCL grouped send/recv on the plan's stream (library-owned communicator)"
                                  if dd.world > 1 else "one rank: local copies"}
    del ins, outs, plan, sc
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def slab_chunks(By, G, req):
    """k-chunks per exchange of a slab plan: csrc/slab.hpp make_geometry (default 4, at most the
    smallest rank's k-range)."""
    from paper_2303_17510_b200.distributed import partition

    kmin = min(b - a for a, b in partition(By, G))
    return max(1, min(req or 4, max(1, kmin)))


def _block(p):
    return p.blockLength()


def _regime(p):
    return p.regime.name


def run_cuda(args):
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29577")
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    dd = Dist(rank, world, local)
    name = default_config(args)
    dims = CONFIGS[name][0]
    t1 = None
    watchdog = None
    if world > 1:
        # a collective that never completes (a lost rank, a wedged link) must not hang the driver: after
        # HCONV_BENCH_TIMEOUT seconds rank 0 prints an error line and every rank exits non-zero
        import threading

        def bail():
            if rank == 0:
                print(json.dumps({"metric": "complex128 dealiased-convolution output points/s", "value": None,
                                  "n_gpus": world, "error": "multi-GPU run timed out", "config": config_dict(name, world)}),
                      flush=True)
            os._exit(3)

        watchdog = threading.Timer(float(os.environ.get("HCONV_BENCH_TIMEOUT", "1500")), bail)
        watchdog.daemon = True
        watchdog.start()
    if world > 1 and dims > 1 and not args.no_t1:
        # T_1: the same global problem on one GPU (rank 0 alone, the single-device path)
        if rank == 0:
            solo = measure(name, argparse.Namespace(**{**vars(args), "slab": False}), Dist(0, 1, local), False)
            t1 = solo["ms_per_step"]
        dd.barrier()
    slab_error = None
    try:
        m = measure(name, args, dd, True)
    except Exception as e:  # noqa: BLE001 -- N > 1: a failing slab path must not lose the run
        if not (world > 1 and dims > 1) or args.config:
            raise
        # every rank fails the same way (the exchange is collective): report the sharded 1D
        # configuration as the headline instead, with the slab error on the line
        slab_error = repr(e)[:300]
        name, dims, t1 = "c2", 1, None
        import torch

        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        m = measure(name, args, dd, True)
    others = {}
    if not args.single:
        extra = ["c1", "c3", "c4", "c5", "c2"] if world == 1 else ["c4", "c2"]
        for o in extra:
            if o == name:
                continue
            try:
                r = measure(o, args, dd, False)
                others[o] = {k: r[k] for k in ("value", "ms_per_step", "plan", "kernel", "input_sets")}
                others[o]["roofline_frac"] = r["roofline"]["frac"]
                others[o]["north_star_frac"] = r["roofline"]["north_star_frac"]
                others[o]["ncu_traffic"] = r["roofline"]["traffic"]
                others[o]["algorithmic_bytes"] = r["roofline"]["algorithmic"]["bytes"]
                others[o]["e2e"] = r["e2e"]["value"]
                others[o]["scaling"] = "weak" if CONFIGS[o][0] == 1 else "strong"
                if "exchange" in r:
                    others[o]["exchange"] = r["exchange"]
            except Exception as e:  # noqa: BLE001 -- a side config must not lose the headline line
                others[o] = {"error": repr(e)[:300]}
    if watchdog is not None:
        watchdog.cancel()
    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    slab = dims > 1 and world > 1
    line = {
        "metric": "complex128 dealiased-convolution output points/s",
        "value": m["value"], "unit": "points/s", "n_gpus": world, "steps": m["steps"], "warmup": m["warmup"],
        "ms_per_step": m["ms_per_step"], "higher_is_better": True, "scaling": "strong" if dims > 1 else "weak",
        "vs_baseline": None, "dtype": "complex128 (f64)",
        "data": "synthetic (counter-based uniform[-1,1], seeds 1..sets; " +
                ("x-slabs of one global problem)" if slab else "each rank its own batch slice)" if dims == 1 else "one global problem)"),
        "config": config_dict(name, world),
        "parallelism": (f"x-slabs over {world} GPUs, NCCL exchanges inside the library" if slab
                        else f"dp{world} (independent batches)" if dims == 1 else "one GPU"),
        "details": {k: m[k] for k in ("plan", "kernel", "launch", "input_sets")},
        "roofline": m["roofline"], "clocks": m.get("clocks"), "e2e": m["e2e"], "gpu_launches": m["gpu_launches"],
    }
    if "exchange" in m:
        line["exchange"] = m["exchange"]
    if slab_error:
        line["slab_error"] = slab_error
    if t1 is not None:
        line["strong_scaling"] = {"t1_ms": t1, "tN_ms": m["ms_per_step"], "N": world,
                                  "efficiency": t1 / (world * m["ms_per_step"]),
                                  "t1_how": "the same problem on rank 0's GPU alone (single-device path), same run"}
    if others:
        line["configs"] = others
    if world == 1 and not args.no_cpu:
        try:
            arm = CpuArm(name)  # the CPU path's own tuned m (the GPU plan's m may not suit the CPU)
            arm.size_for(15.0)
            v, dt = arm.run()
            line["cpu_baseline"] = {"value": v, "unit": "points/s", "cores": arm.threads, "kind": "port",
                                    "sample": arm.sample(dt)}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": "points/s", "cores": os.cpu_count(), "kind": "port",
                                    "sample": repr(e)[:200]}
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def self_launch(args) -> int:
    """--gpus N > 1 without a torchrun environment: run this script under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1); rank 0's line is the output."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS), help="default: c2 at 1 GPU, c5 (slabs) above")
    ap.add_argument("--m", default=None, help="force subtransform size(s): one value or one per axis, comma separated")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--single", action="store_true", help="only the headline configuration (no 'configs' sub-object)")
    ap.add_argument("--slab", action="store_true", help="2D/3D: run the x-slab decomposition even on one rank")
    ap.add_argument("--chunks", type=int, default=0, help="slab: k-chunks per exchange (0 = library default)")
    ap.add_argument("--no-t1", action="store_true", help="slabs over N > 1 GPUs: skip the one-GPU T_1 measurement")
    ap.add_argument("--no-graph", action="store_true", help="issue every step through the API instead of a CUDA graph")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "cuda":
        sys.exit(self_launch(args))
    if args.launch_check:  # test hook: the rank layout bench.py runs with (no GPU work)
        line = json.dumps({"rank": rank, "world": world, "local": local, "config": default_config(args)}) + "\n"
        sys.stdout.flush()
        os.write(1, line.encode())  # one write per rank: the ranks share the launcher's pipe
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_cuda(args)


if __name__ == "__main__":
    main()
