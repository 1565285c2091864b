"""The slab plan (hconv_desc.slab, csrc/slab.hpp) of the CUDA library on one GPU -- the y-axis
passes in k-major layout, the placement copies, the chunked schedule over two streams and the
inner batched subconvolutions -- against the single-device convolve_nd on the same seeded
inputs, with each exchange flavour at one rank: none (local copy), the library's own NCCL
communicator (binding, comm init, grouped calls) and the torch.distributed callback on the
library's communication stream.  Multi-rank index arithmetic: tests/test_distributed_cpu.py."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    "2d_complex": [(256, 511, 256, 0), (192, 383, 128, 0)],
    "3d_hermitian": [(63, 94, 32, 1), (63, 94, 48, 1), (63, 94, 32, 2)],
    "3d_complex": [(40, 79, 40, 0), (48, 95, 32, 0), (24, 47, 24, 0)],
    "2d_tiny": [(2, 3, 2, 0), (4, 7, 2, 0)],  # at three ranks some hold no x rows / no k rows
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(port, q):
    import torch
    import torch.distributed as dist

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        import sys
        from pathlib import Path

        repo = Path(__file__).resolve().parents[1]
        sys.path.insert(0, str(repo))
        sys.path.insert(0, str(repo / "tests"))
        from oracle_lib import rel_l2
        from paper_2303_17510_b200 import hconv
        from paper_2303_17510_b200.distributed import NcclComm, SlabAxis, SlabConvND

        res = {}
        comm = NcclComm()
        for name, axes in CASES.items():
            shape = tuple((L + 1) // 2 if s == 2 else L for L, M, m, s in axes)
            f = torch.empty(shape, dtype=torch.complex128, device="cuda")
            g = torch.empty_like(f)
            hconv.fill_uniform(f, 2, 0)
            hconv.fill_uniform(g, 2, 1)
            if axes[-1][3] == 2:
                hconv.hermitian_symmetrize_boundary(f, [a[0] for a in axes])
                hconv.hermitian_symmetrize_boundary(g, [a[0] for a in axes])
            plan = hconv.ConvPlanND([hconv.AxisSpec(L, M, m, hconv.Symmetry(s)) for L, M, m, s in axes])
            ref = hconv.convolve_nd([f, g], plan.mult, plan, out=torch.empty_like(f))[0].cpu().numpy()
            for flavour, chunks in (("none", 0), ("nccl", 3), ("torch", 2)):
                sc = SlabConvND([SlabAxis(*a) for a in axes], comm=comm if flavour == "nccl" else flavour,
                                chunks=chunks)
                h = sc.convolve([f.clone(), g.clone()])[0]
                torch.cuda.synchronize()
                res[f"{name}_{flavour}"] = rel_l2(h.cpu().numpy(), ref)
                assert sc.workspace_bytes() > 0
                del sc
        del comm
        q.put((res, None))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback

        q.put((None, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_slab_single_rank_nccl_matches_convolve_nd(cuda):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_free_port(), q))
    p.start()
    res, tb = q.get(timeout=600)
    p.join(timeout=60)
    assert tb is None, tb
    for name, err in res.items():
        assert err <= 1e-12, (name, err)


def _worker_multi(rank, world, port, q):
    """rank of a world-`world` gloo group, every rank on cuda:0: the CUDA library's slab driver
    with real kernels and a host-staged exchange callback (no kernel waits on another rank: the
    exchange is a synchronous host all-to-all), against the single-device convolve_nd."""
    import torch
    import torch.distributed as dist

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        from pathlib import Path

        repo = Path(__file__).resolve().parents[1]
        sys.path.insert(0, str(repo))
        sys.path.insert(0, str(repo / "tests"))
        from oracle_lib import rel_l2
        from paper_2303_17510_b200 import hconv
        from paper_2303_17510_b200.distributed import SlabAxis, SlabConvND

        res = {}
        for name, axes in CASES.items():
            shape = tuple((L + 1) // 2 if s == 2 else L for L, M, m, s in axes)
            f = torch.empty(shape, dtype=torch.complex128, device="cuda")
            g = torch.empty_like(f)
            hconv.fill_uniform(f, 4, 0)
            hconv.fill_uniform(g, 4, 1)
            if axes[-1][3] == 2:
                hconv.hermitian_symmetrize_boundary(f, [a[0] for a in axes])
                hconv.hermitian_symmetrize_boundary(g, [a[0] for a in axes])
            plan = hconv.ConvPlanND([hconv.AxisSpec(L, M, m, hconv.Symmetry(s)) for L, M, m, s in axes])
            ref = hconv.convolve_nd([f, g], plan.mult, plan, out=torch.empty_like(f))[0]
            for chunks in (0, 3):
                sc = SlabConvND([SlabAxis(*a) for a in axes], comm="torch", chunks=chunks)
                x0, nx = sc.x0, sc.nx
                h = sc.convolve([f[x0:x0 + nx].clone(), g[x0:x0 + nx].clone()])[0]
                torch.cuda.synchronize()
                res[f"{name}_c{chunks}"] = rel_l2(h.cpu().numpy(), ref[x0:x0 + nx].cpu().numpy()) if nx else 0.0
                del sc
        q.put((rank, res, None))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, None, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_multi_rank_cuda_kernels_host_exchange(cuda, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_multi, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, res, tb in results:
        assert tb is None, tb
        for name, err in res.items():
            assert err <= 1e-12, (rank, name, err)
