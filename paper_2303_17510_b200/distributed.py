"""Slab-decomposed 2D/3D dealiased convolution over several GPUs, through the C ABI.

The reference has no distributed code (SPEC.md:512 lists MPI decomposition as a non-goal); this
is the multi-GPU extension the north star asks for.  The decomposition itself -- index
arithmetic, buffers, the schedule and the exchanges -- is native C++ behind the C ABI
(``hconv_desc.slab``, include/hconv.h; driver csrc/slab.hpp): the global arrays [x][y] (2D) or
[x][y][z] (3D, z innermost) are split into x-slabs, the outer padded FFT runs along the locally
complete axis y, and per y residue two all-to-alls bring complete x-lines to every rank for the
(d-1)-D subconvolutions and back.  This module only
  * creates the plan (every m given; ``choose_sizes`` tunes on rank 0 and broadcasts),
  * provides the exchange: an NCCL communicator the library drives itself (CUDA library, G > 1:
    grouped ncclSend/ncclRecv on its own stream, chunk by chunk against the subconvolutions), or
    a torch.distributed all-to-all callback (gloo in the CPU tests, where the library is the
    oracle exporting the same ABI over host memory -- test infrastructure only).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _abi


def partition(n: int, parts: int) -> list[tuple[int, int]]:
    """Balanced contiguous split of range(n), the one csrc/slab.hpp uses (511 = 7*64 + 63)."""
    base, extra = divmod(n, parts)
    out, lo = [], 0
    for g in range(parts):
        hi = lo + base + (1 if g < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


@dataclass
class SlabAxis:
    L: int
    M: int
    m: int
    symmetry: int = _abi.COMPLEX


def _view(ptr: int, count: int, device: torch.device) -> torch.Tensor:
    """complex128 tensor over `count` elements at a raw address (no copy)."""
    if count == 0:
        return torch.empty(0, dtype=torch.complex128, device=device)
    if device.type == "cuda":
        from .hconv import _CudaArray

        return torch.as_tensor(_CudaArray(ptr, count, False), device=device)
    arr = np.ctypeslib.as_array(C.cast(C.c_void_p(ptr), C.POINTER(C.c_double)), (2 * count,))
    return torch.from_numpy(arr.view(np.complex128))


class _TorchExchange:
    """hconv_exchange_fn over torch.distributed: the per-peer segments are packed into one
    contiguous buffer for all_to_all_single (gloo has no list all-to-all) and unpacked at their
    displacements.  CUDA pointers: ordered on the library's communication stream."""

    def __init__(self, group, device: torch.device):
        self.group = group
        self.device = device
        self.G = dist.get_world_size(group)
        # a gloo group cannot exchange CUDA tensors: stage device segments through host memory
        self.host_staged = device.type == "cuda" and dist.get_backend(group) == "gloo"
        self.cb = _abi.ExchangeFn(self._fn)
        self.error: Optional[str] = None

    def _fn(self, send, sc, sd, recv, rc, rd, user, stream):
        try:
            G = self.G
            sc_, sd_, rc_, rd_ = ([int(a[h]) for h in range(G)] for a in (sc, sd, rc, rd))
            ctx = (torch.cuda.stream(torch.cuda.ExternalStream(stream, device=self.device))
                   if self.device.type == "cuda" else _null())
            with ctx:
                src = _view(send, max((d + c for d, c in zip(sd_, sc_)), default=0), self.device)
                dst = _view(recv, max((d + c for d, c in zip(rd_, rc_)), default=0), self.device)
                packed = torch.cat([src[d:d + c] for d, c in zip(sd_, sc_)]) if sum(sc_) else src[:0].clone()
                xdev = torch.device("cpu") if self.host_staged else self.device
                out = torch.empty(sum(rc_), dtype=torch.complex128, device=xdev)
                dist.all_to_all_single(torch.view_as_real(out).view(-1), torch.view_as_real(packed.to(xdev)).view(-1),
                                       [2 * c for c in rc_], [2 * c for c in sc_], group=self.group)
                out = out.to(self.device)
                off = 0
                for d, c in zip(rd_, rc_):
                    dst[d:d + c].copy_(out[off:off + c])
                    off += c
            return 0
        except Exception as e:  # noqa: BLE001 -- reported as HCONV_NCCL_ERROR by the library
            self.error = repr(e)
            return 1


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class NcclComm:
    """An NCCL communicator of the CUDA library over the ranks of a torch.distributed group
    (unique id from rank 0, broadcast through the group)."""

    def __init__(self, group=None, device: Optional[torch.device] = None):
        from . import hconv

        self.lib = hconv.lib()
        rank, G = dist.get_rank(group), dist.get_world_size(group)
        dev = device or torch.device("cuda", torch.cuda.current_device())
        uid = (C.c_char * 128)()
        if rank == 0:
            _abi.check(self.lib, self.lib.hconv_nccl_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (C.c_char * 128).from_buffer_copy(obj[0])
        self.h = C.c_void_p()
        _abi.check(self.lib, self.lib.hconv_nccl_comm_init(uid, G, rank, dev.index or 0, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.hconv_nccl_comm_destroy(self.h)
            self.h = None


class SlabConvND:
    """x-slab plan of a 2D complex or 3D (complex or Hermitian) convolution (hconv_desc.slab).

    axes: [x, y] or [x, y, z], every m given; Hermitian mode = z Hermitian (x, y centered,
    PAPER.md:639-642).  lib: a library exporting include/hconv.h -- the CUDA library (default;
    device slabs) or, in the CPU tests, the oracle (host slabs).  comm: "nccl" (the library's own
    NCCL communicator; CUDA, default when G > 1) or an NcclComm to share, "torch" (all-to-all
    callback over `group`), "none" (one rank: the exchange is a local copy; default at G = 1).
    mult: None = builtin product (A = 2, B = 1), else an hconv.MultOperator.
    """

    def __init__(self, axes: Sequence[SlabAxis], lib: Optional[C.CDLL] = None, group=None, mult=None,
                 comm: str = "auto", chunks: int = 0, device: Optional[torch.device] = None):
        if len(axes) not in (2, 3):
            raise ValueError("slab decomposition is for 2D and 3D convolutions")
        self.axes = list(axes)
        self.group = group
        self.G = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if lib is None:
            from . import hconv

            lib = hconv.lib()
        self.lib = lib
        self.cuda = lib.hconv_backend() == b"cuda-sm_100a"
        self.device = (device or torch.device("cuda", torch.cuda.current_device())) if self.cuda else torch.device("cpu")
        self.A, self.B = (2, 1) if mult is None else (mult.A, mult.B)
        self._comm = None
        self._xch = None
        s = _abi.Slab()
        s.rank, s.nranks, s.chunks = self.rank, self.G, chunks
        if comm == "auto":
            comm = ("nccl" if self.cuda else "torch") if self.G > 1 else "none"
        if isinstance(comm, NcclComm) or comm == "nccl":
            if not self.cuda:
                raise ValueError("NCCL exchange needs the CUDA library")
            self._comm = comm if isinstance(comm, NcclComm) else NcclComm(group, self.device)
            s.nccl_comm = self._comm.h
        elif comm == "torch":
            self._xch = _TorchExchange(group, self.device)
            s.exchange = C.cast(self._xch.cb, C.c_void_p)
        elif comm != "none" or self.G > 1:
            raise ValueError(f"comm must be 'nccl', 'torch', an NcclComm (or 'none' at one rank), not {comm!r}")
        self._slab = s
        d = _abi.Desc()
        d.dims = len(axes)
        for k, a in enumerate(axes):
            d.axis[k] = _abi.Axis(a.L, a.M, a.m, a.symmetry)
        d.A, d.B, d.C, d.dist = self.A, self.B, 1, 0
        d.device = (self.device.index or 0) if self.cuda else 0
        self._mult_keep = None
        if mult is None or mult.kind == _abi.MULT_PRODUCT:
            d.mult = _abi.MULT_PRODUCT
        else:
            d.mult = mult.kind
            fn, self._mult_keep = mult._native(host=not self.cuda)
            d.mult_fn = fn
        d.slab = C.cast(C.pointer(s), C.c_void_p)
        h = C.c_void_p()
        _abi.check(lib, lib.hconv_plan_create(C.byref(d), C.byref(h)))
        self.h = h
        x0, nx = C.c_size_t(), C.c_size_t()
        _abi.check(lib, lib.hconv_plan_slab(h, C.byref(x0), C.byref(nx)))
        self.x0, self.nx = x0.value, nx.value
        herm = axes[-1].symmetry == _abi.HERMITIAN
        self.data = [((a.L + 1) // 2 if (herm and k == len(axes) - 1) else a.L) for k, a in enumerate(axes)]
        self.xs = partition(self.data[0], self.G)

    def local_shape(self) -> tuple[int, ...]:
        return (self.nx, *self.data[1:])

    def params(self, axis: int):
        """the axis' PlanParams (hconv.PlanParams: m, p, q, n, blockLength(), ...)."""
        from .hconv import PlanParams

        p = _abi.Params()
        _abi.check(self.lib, self.lib.hconv_plan_params(self.h, axis, C.byref(p)))
        return PlanParams._from_c(p)

    def workspace_bytes(self) -> int:
        return int(self.lib.hconv_plan_workspace_bytes(self.h))

    def convolve(self, inputs: Sequence[torch.Tensor], out: Optional[Sequence[torch.Tensor]] = None) -> list[torch.Tensor]:
        """inputs: this rank's x-slabs (local_shape()) of the A inputs; returns the B output slabs
        (by default written over the first B inputs, the reference's in-place convention)."""
        if isinstance(inputs, torch.Tensor):
            raise TypeError("pass a sequence of input slabs")
        if len(inputs) != self.A:
            raise ValueError(f"expected {self.A} input slabs")
        for t in inputs:
            if tuple(t.shape) != self.local_shape() or t.dtype != torch.complex128 or not t.is_contiguous():
                raise ValueError(f"expected contiguous complex128 slabs of shape {self.local_shape()}")
            if t.device.type != self.device.type:
                raise ValueError(f"slabs must live on {self.device.type}")
        outs = list(inputs[:self.B]) if out is None else list(out)
        if len(outs) != self.B:
            raise ValueError(f"expected {self.B} output slabs")
        i = (C.c_void_p * self.A)(*[t.data_ptr() for t in inputs])
        o = (C.c_void_p * self.B)(*[t.data_ptr() for t in outs])
        stream = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream) if self.cuda else None
        st = self.lib.hconv_convolve(self.h, i, o, stream)
        if st != _abi.OK and self._xch is not None and self._xch.error:
            raise RuntimeError(f"slab exchange failed: {self._xch.error}")
        _abi.check(self.lib, st)
        return outs

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.hconv_plan_destroy(self.h)
            self.h = None


def choose_sizes(axes: Sequence[tuple[int, int, int]], group=None, device: Optional[torch.device] = None) -> list[int]:
    """The device-timed planner's m per axis (tune_nd on rank 0's GPU over the whole problem),
    broadcast so that every rank builds the same plan (the y blocks must agree).
    axes: [(L, M, symmetry)]."""
    from . import hconv

    chosen = [None]
    if not dist.is_initialized() or dist.get_rank(group) == 0:
        plan = hconv.ConvPlanND([hconv.AxisSpec(L, M, None, hconv.Symmetry(s)) for L, M, s in axes],
                                device=(device.index or 0) if device is not None else 0)
        chosen = [[p.m for p in plan.params]]
        del plan
    if dist.is_initialized():
        dist.broadcast_object_list(chosen, src=0, group=group)
    return list(chosen[0])
