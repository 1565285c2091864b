#!/usr/bin/env python3
"""Benchmark of the hybrid-dealiased convolution path on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[1], the config the metric is quoted on): 1D complex binary
convolution, L = 6000, M = 11999, batch 4096 per GPU (weak scaling: the batch is sharded, no
collective on the data path), complex128 inputs uniform[-1,1] from the counter-based generator,
m/p/q chosen by the device-timed planner.  A step is one convolution of the whole batch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference] [--config c1..c5]

--impl reference times the reference's CPU path on the host cores: the reference's own code
cannot be built (FFTW++/FFTW absent), so this is the CPU restatement in oracle/
(kind "port"), rank 0 only, on a bounded sample of copies per step.
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


# ------------------------------------------------------------------ CPU arm ------
def launches_per_step(params):
    """kernels one step launches: 1D = 1 fused conv; N-D = per outer residue A forward + inner + 1 backward."""
    if len(params) == 1:
        return 1
    inner = launches_per_step(params[1:])
    return params[0].n * (A + inner + 1)


# candidate subtransform sizes of the CPU baseline's own tuning probe (hybrid, explicit, pow2)
CPU_CANDIDATES = {"c1": [256, 512, 1024, 2048], "c2": [1024, 1536, 2000, 2048, 3000, 3072, 4096, 6000, 6144, 12000],
                  "c3": [2048, 4096, 8192, 12288]}


class CpuArm:
    """Oracle (CPU restatement, TEST INFRASTRUCTURE) on a bounded sample of the 1D workload:
    a probe sizes the sample, then each call convolves `rows` copies of the batch."""

    def __init__(self, name, m=None, threads=None):
        sys.path.insert(0, str(REPO / "tests"))
        from oracle_lib import Oracle

        self.o = Oracle()
        self.threads = threads or os.cpu_count()
        self.o.lib.oracle_set_threads(self.threads)
        dims, axes, self.C, shape, n_out = config_sizes(name)
        if dims != 1:
            raise SystemExit("CPU baseline is timed on the 1D configs (N-D: tools/bench_all.py)")
        self.L, self.M, self.s = axes[0]
        self.S = shape[0]
        probe = max(self.threads, 8)
        self.rows = probe
        if m:
            self.m = m
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
        self.rows = int(min(self.C, max(self.threads, seconds / max(self.per_row, 1e-9))))

    def run(self):
        f = self.o.uniform(1, 0, self.rows * self.S).reshape(self.rows, self.S)
        g = self.o.uniform(1, 1, self.rows * self.S).reshape(self.rows, self.S)
        t0 = time.perf_counter()
        self.o.convolve([(self.L, self.M, self.m, self.s)], f, g, C_=self.rows)
        dt = time.perf_counter() - t0
        return self.rows * self.S / dt, dt

    def sample(self, dt):
        return f"{self.rows} of {self.C} copies per step (m={self.m}), {dt:.2f} s per step"


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    name = args.config
    dims, axes, C_, shape, n_out = config_sizes(name)
    arm = CpuArm(name, int(str(args.m).split(",")[0]) if args.m else None)
    arm.size_for(max(0.5, 120.0 / (args.steps + args.warmup)))  # whole run ~2 minutes
    vals, dts = [], []
    for i in range(args.warmup + args.steps):
        v, dt = arm.run()
        if i >= args.warmup:
            vals.append(v)
            dts.append(dt)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "complex128 dealiased-convolution output points/s", "value": value,
        "unit": "points/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": n_out / value * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "complex128 (f64)", "data": "synthetic (counter-based uniform[-1,1], seed 1)",
        "config": {"workload": WORKLOAD[name], "config": name},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": arm.threads, "kind": "port",
                         "sample": arm.sample(statistics.median(dts)) +
                         "; CPU restatement (oracle/), the reference's FFTW++/FFTW path is not buildable here"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm ------
def run_cuda(args):
    import torch

    from paper_2303_17510_b200 import hconv

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.slab:
        import torch.distributed as dist

        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29577")
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    name = args.config
    dims, axes, C_, shape, n_out = config_sizes(name)
    stream = torch.cuda.current_stream()

    # plan (planner runs here, outside the timed region); --m: one size for every axis or a list
    ms = [None] * dims
    if args.m:
        vals = [int(x) for x in str(args.m).split(",")]
        ms = vals if len(vals) == dims else [vals[0]] * dims
    # 2D/3D over several GPUs: x-slabs, NCCL all-to-all (strong scaling); --slab forces the slab
    # path at one rank (exercises the decomposition on a single GPU)
    slab = dims > 1 and (world > 1 or args.slab)
    if dims == 1:
        L, M, s = axes[0]
        plan = hconv.Conv1dPlan(L, M, ms[0], hconv.Symmetry(s), C_=C_, device=local)
        params = [plan.params]
    else:
        # the planner runs on rank 0 and every rank uses its choice (the y blocks must agree)
        chosen = [None]
        if rank == 0 or not slab:
            plan = hconv.ConvPlanND([hconv.AxisSpec(L, M, mk, hconv.Symmetry(s)) for (L, M, s), mk in zip(axes, ms)],
                                    device=local)
            chosen = [[p.m for p in plan.params]]
        if slab:
            import torch.distributed as dist

            dist.broadcast_object_list(chosen, src=0)
            plan = hconv.ConvPlanND([hconv.AxisSpec(L, M, mk, hconv.Symmetry(s)) for (L, M, s), mk in zip(axes, chosen[0])],
                                    device=local)
        params = plan.params
    full_shape = (C_, *shape) if dims == 1 else tuple(shape)
    f = torch.empty(full_shape, dtype=torch.complex128, device=dev)
    g = torch.empty_like(f)
    first = rank * f.numel() if not slab else 0  # 1D: each rank owns its own slice of the global batch
    hconv.fill_uniform(f, 1, 0, first)
    hconv.fill_uniform(g, 1, 1, first)
    if dims == 3:
        hconv.hermitian_symmetrize_boundary(f, [L for (L, M, s) in axes])
        hconv.hermitian_symmetrize_boundary(g, [L for (L, M, s) in axes])
    sc = None
    if slab:
        from paper_2303_17510_b200.distributed import SlabAxis, SlabConvND, cuda_backend

        sc = SlabConvND([SlabAxis(L, M, p.m, s) for (L, M, s), p in zip(axes, params)], cuda_backend(dev))
        x0, x1 = sc.xs[rank]
        f, g = f[x0:x1].clone(), g[x0:x1].clone()  # this rank's x-slabs of the global arrays
        torch.cuda.empty_cache()
    out = torch.empty_like(f)

    def step():
        if dims == 1:
            hconv.convolve([f, g], plan.mult, plan, out=out)
        elif slab:
            sc.convolve([f, g], out=[out])
        else:
            hconv.convolve_nd([f, g], plan.mult, plan, out=out)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier(device_ids=[local])

    if not slab and not args.no_graph:
        # the step's kernels captured once in a CUDA graph (warm-up and capture outside the timed
        # region); each timed step replays the whole convolution of the batch
        cap = hconv.CapturedConvolution([f, g], plan.mult, plan, out=out)
        step = cap  # noqa: F811
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    # 1D: every rank convolves its own batch (weak scaling); slabs: the ranks share one problem
    value = (1 if slab else world) * n_out * args.steps / (ms * 1e-3)

    # e2e through the public host-buffer API (hconv.convolve_host, the reference's calling
    # convention): every step copies both inputs from pinned host memory to the device and the
    # result back (1D: in chunks, copies and compute overlapped on three streams)
    hf = f.cpu().pin_memory()
    hg = g.cpu().pin_memory()
    ho = torch.empty_like(hf).pin_memory()

    def step_host():
        if slab:  # host slabs in, device convolution, host slab out
            fd, gd = hf.to(dev, non_blocking=True), hg.to(dev, non_blocking=True)
            ho.copy_(sc.convolve([fd, gd])[0], non_blocking=True)
            torch.cuda.current_stream().synchronize()
        else:
            hconv.convolve_host([hf, hg], plan.mult, plan, out=ho)

    for _ in range(2):
        step_host()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e2e_steps = max(1, min(args.steps, 5))
    # the host call is synchronous: events on the (idle) current stream bracket whole calls
    e0.record(stream)
    for _ in range(e2e_steps):
        step_host()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = (1 if slab else world) * n_out * e2e_steps / (e2e_ms * 1e-3)

    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    hbm, src_h, fp64, src_f = peaks()
    nbytes, flops = algorithmic(name)
    if slab:  # per-GPU share of the one global problem (the roofline is per GPU)
        nbytes, flops = nbytes / world, flops / world
    t_s = ms_step * 1e-3
    achieved_tf = flops / t_s / 1e12
    t_roof = max(nbytes / (hbm * 1e9), flops / (fp64 * 1e12))
    traffic = None
    tp = REPO / "profiles" / f"r01_{name}_ncu_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get("dram_bytes_per_launch")
    launches = args.steps * launches_per_step(params)
    if slab:  # per y residue: A forward + the batched subconvolutions + B backward (torch copies not counted)
        launches = args.steps * params[1].n * (A + launches_per_step([params[0]] + params[2:]) + B)
    line = {
        "metric": "complex128 dealiased-convolution output points/s",
        "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong" if slab else "weak", "vs_baseline": None,
        "dtype": "complex128 (f64)",
        "data": "synthetic (counter-based uniform[-1,1], seed 1; " + ("x-slabs of one global problem)" if slab else "each rank its own batch slice)"),
        "config": {
            "workload": WORKLOAD[name], "config": name, "batch_per_gpu": C_, "global_batch": C_ * (1 if slab else world),
            "parallelism": (f"x-slabs over {world} GPUs, NCCL all-to-all per y residue" if slab else f"dp{world} (independent batches)"),
            "launch": "direct API calls" if (slab or args.no_graph) else "CUDA graph replay of the API call (captured once)",
            "plan": [dict(m=p.m, p=p.p, q=p.q, n=p.n, block=p.blockLength(), regime=p.regime.name) for p in params],
            "kernel": plan.kernel(len(params) - 1),
            "l2": "inputs+output larger than L2 (3 x 393 MB vs 126 MB)" if name == "c2" else "see config",
        },
        "roofline": {
            "bound": "fp64", "achieved": achieved_tf, "peak": fp64, "unit": "TFLOP/s", "frac": achieved_tf / fp64,
            "traffic": traffic, "peak_source": src_f,
            "hbm": {"achieved": nbytes / t_s / 1e9, "peak": hbm, "unit": "GB/s", "frac": nbytes / t_s / 1e9 / hbm,
                    "peak_source": src_h},
            "north_star_frac": t_roof / t_s,
            "algorithmic": {"bytes": nbytes, "flops": flops},
        },
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": 2 * f.numel() * 16,
                "d2h_bytes_per_step": out.numel() * 16, "steps": e2e_steps},
        "gpu_launches": launches,
    }
    if world == 1 and not args.no_cpu:
        try:
            arm = CpuArm(name)  # the CPU path's own tuned m (the GPU plan's m may not suit the CPU)
            arm.size_for(15.0)
            v, dt = arm.run()
            line["cpu_baseline"] = {"value": v, "unit": "points/s", "cores": arm.threads, "kind": "port",
                                    "sample": arm.sample(dt)}
        except SystemExit as e:
            line["cpu_baseline"] = {"value": None, "unit": "points/s", "cores": os.cpu_count(), "kind": "port", "sample": str(e)}
    print(json.dumps(line), flush=True)
    if world > 1 or args.slab:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--m", default=None, help="force subtransform size(s): one value or one per axis, comma separated")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--slab", action="store_true", help="2D/3D: run the x-slab decomposition even on one rank")
    ap.add_argument("--no-graph", action="store_true", help="issue every step through the API instead of a CUDA graph")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_cuda(args)


if __name__ == "__main__":
    main()
