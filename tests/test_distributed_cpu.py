"""Multi-rank slab decomposition on CPU: world_size 2 and 3 over gloo.  The plan is the C ABI's
slab plan (hconv_desc.slab) of the oracle library, which runs the product's native driver
(paper_2303_17510_b200/csrc/slab.hpp: index arithmetic, chunked exchanges, placement copies)
over host memory with the oracle's padded FFTs and a torch.distributed all-to-all callback;
checked slab by slab against the single-process oracle convolve_nd."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = {
    "2d_complex": [(6, 11, 3, 0), (5, 9, 2, 0)],
    "2d_complex_odd": [(7, 13, 7, 0), (9, 17, 4, 0)],
    "3d_complex": [(5, 9, 3, 0), (4, 7, 2, 0), (3, 5, 3, 0)],
    "3d_hermitian": [(7, 11, 4, 1), (7, 11, 2, 1), (7, 11, 4, 2)],
    "3d_hermitian_inner": [(9, 14, 2, 1), (9, 14, 3, 1), (9, 14, 2, 2)],
    # more ranks than x rows / y spectral rows: some ranks hold no slab rows or no k-rows
    "2d_tiny": [(2, 3, 2, 0), (4, 7, 2, 0)],
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        from pathlib import Path

        repo = Path(__file__).resolve().parents[1]
        sys.path.insert(0, str(repo))
        sys.path.insert(0, str(repo / "tests"))
        from oracle_lib import Oracle, rel_l2
        from paper_2303_17510_b200.distributed import SlabAxis, SlabConvND

        o = Oracle()
        o_ = o

        def o_ref(oo, axes, x, y):
            return oo.convolve(axes, x, y)

        axes = CASES[case]
        herm = axes[-1][3] == 2
        shape = [((L + 1) // 2 if s == 2 else L) for (L, M, m, s) in axes]
        rng = np.random.default_rng(11)
        f = rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)
        g = rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)
        if herm:
            f = o.symmetrize([a[0] for a in axes], f)
            g = o.symmetrize([a[0] for a in axes], g)
        ref = o.convolve(axes, f, g)
        err = 0.0
        for chunks in (0, 1, 3):
            sc = SlabConvND([SlabAxis(L, M, m, s) for (L, M, m, s) in axes], lib=o.lib, chunks=chunks)
            x0, x1 = sc.xs[rank]
            assert (sc.x0, sc.nx) == (x0, x1 - x0)
            fl = torch.from_numpy(f[x0:x1].copy())
            gl = torch.from_numpy(g[x0:x1].copy())
            h = sc.convolve([fl, gl])[0].numpy()  # in place over fl
            err = max(err, rel_l2(h, ref[x0:x1]))
        # a general A = 2 -> B = 3 operator through the same decomposition
        from paper_2303_17510_b200 import hconv

        def pairs(b, real):
            f0, f1 = b[0].clone(), b[1].clone()
            b[0].copy_(f0 * f0)
            b[1].copy_(f0 * f1)
            b[2].copy_(f1 * f1)

        op = hconv.mult_operator(2, 3, pairs)
        sc3 = SlabConvND([SlabAxis(L, M, m, s) for (L, M, m, s) in axes], lib=o.lib, mult=op)
        fl = torch.from_numpy(f[x0:x1].copy())
        gl = torch.from_numpy(g[x0:x1].copy())
        outs = sc3.convolve([fl, gl], out=[torch.empty_like(fl) for _ in range(3)])
        for o, (x, y) in zip(outs, [(f, f), (f, g), (g, g)]):
            err = max(err, rel_l2(o.numpy(), o_ref(o_, axes, x, y)[x0:x1]))
        q.put((rank, err, None))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, None, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", sorted(CASES))
def test_slab_decomposition_matches_oracle(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, tb in results:
        assert tb is None, tb
        assert err <= 1e-12, (rank, err)


def test_partition_uneven():
    from paper_2303_17510_b200.distributed import partition

    parts = partition(511, 8)
    assert parts[0] == (0, 64) and parts[-1] == (448, 511)
    assert sum(b - a for a, b in parts) == 511


def test_slab_single_rank_without_process_group(oracle):
    """G = 1 needs no exchange: the plan's own segment is a local copy."""
    from oracle_lib import rel_l2
    from paper_2303_17510_b200.distributed import SlabAxis, SlabConvND

    axes = [(7, 11, 4, 1), (7, 11, 2, 1), (7, 11, 4, 2)]
    shape = [((L + 1) // 2 if s == 2 else L) for (L, M, m, s) in axes]
    rng = np.random.default_rng(3)
    f = oracle.symmetrize([7, 7, 7], rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape))
    g = oracle.symmetrize([7, 7, 7], rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape))
    sc = SlabConvND([SlabAxis(*a) for a in axes], lib=oracle.lib, chunks=2)
    h = sc.convolve([torch.from_numpy(f.copy()), torch.from_numpy(g.copy())], out=[torch.zeros(shape, dtype=torch.complex128)])[0]
    assert rel_l2(h.numpy(), oracle.convolve(axes, f, g)) <= 1e-12


def test_slab_plan_errors(oracle):
    from paper_2303_17510_b200.distributed import SlabAxis, SlabConvND

    with pytest.raises(ValueError):  # m must be given in a slab plan
        SlabConvND([SlabAxis(8, 15, 0), SlabAxis(8, 15, 8)], lib=oracle.lib)
    with pytest.raises(ValueError):  # 1D is not a slab problem
        SlabConvND([SlabAxis(8, 15, 8)], lib=oracle.lib)
