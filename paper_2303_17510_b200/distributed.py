"""Slab-decomposed 2D/3D dealiased convolution over several GPUs.

The reference has no distributed code (SPEC.md:512 lists MPI decomposition as a non-goal); this
is the multi-GPU extension the north star asks for, built on the same C ABI.

Layout: the contiguous arrays [x][y] (2D) or [x][y][z] (3D, z innermost) are split into x-slabs,
rank g owning rows [x0_g, x1_g).  Because a padded FFT needs its whole axis, the OUTER padded
transform runs along y, which every rank holds completely; the sharded axis x becomes an inner
axis after one all-to-all transpose:

  for each residue block r of the y axis (PAPER.md:584-600 with y as the outer axis):
    1. local forward padded y-FFT of the A inputs, ONE strided launch per input
       (hconv_pfft_forward_lines), written k-major: F_a[k][x][z], so the k-block destined for
       rank h is one contiguous run (the all-to-all send buffer needs no packing); each input's
       exchange is issued asynchronously, so it overlaps the next input's forward (and each
       output's exchange the previous output's backward)
    2. all-to-all: rank g receives the spectral y-lines k in [k0_g, k1_g) of every x-slab,
       [h][k][x_h][z], and places them as T_a[k][x][z] with x complete (G slice copies)
    3. the (d-1)-D subconvolutions of all nk spectral lines in ONE batched call
       (hconv_convolve with C = nk; the plan, and with it the multiplication operator, is
       created once); outputs in place in T_b, b < B
    4. all-to-all back: the pieces [h][k][x_g][z] land as W_b[k][x][z] (k-major again)
    5. local inverse padded y-FFT of block r, accumulated into h_b, the last residue scaled by
       1/(q_y m_y) (hconv_pfft_backward_lines)

The multi-D DFT is separable and the inner subconvolutions are pointwise in the y frequency,
so this equals the paper's x-outer recursion numerically.  Exactly (A + B) exchanges per
residue carry L_x x B_y x (inner) values each.  The collective is torch.distributed
all_to_all_single (NCCL over NVLink on GPUs; gloo on CPU in the tests).

The local compute goes through a Backend bound to a library exporting include/hconv.h: the
sm_100a library with CUDA tensors (product), or -- in the CPU tests only -- the oracle with host
tensors, which exercises exactly the same index arithmetic.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import torch
import torch.distributed as dist

from . import _abi


def partition(n: int, parts: int) -> list[tuple[int, int]]:
    """Balanced contiguous split of range(n) (uneven sizes allowed: 511 = 7*64 + 63)."""
    base, extra = divmod(n, parts)
    out, lo = [], 0
    for g in range(parts):
        hi = lo + base + (1 if g < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def _lines(count, nin, d_out, d_in, es) -> _abi.Lines:
    return _abi.Lines(count, nin, d_out, d_in, es)


class _LocalPlan:
    """A convolution plan of the backend's library (owns the operator callback)."""

    def __init__(self, be: "Backend", desc: _abi.Desc, mult):
        self.be = be
        fn, self._keep = (None, None) if mult is None else mult._native(host=be.device.type != "cuda")
        desc.mult_fn = fn
        h = C.c_void_p()
        be._check(be.lib.hconv_plan_create(C.byref(desc), C.byref(h)))
        self.h = h
        self.A, self.B = desc.A, desc.B

    def convolve(self, ins: Sequence[torch.Tensor], outs: Sequence[torch.Tensor]) -> None:
        i = (C.c_void_p * len(ins))(*[t.data_ptr() for t in ins])
        o = (C.c_void_p * len(outs))(*[t.data_ptr() for t in outs])
        self.be._check(self.be.lib.hconv_convolve(self.h, i, o, self.be.stream_fn()))

    def __del__(self):
        if getattr(self, "h", None):
            self.be.lib.hconv_plan_destroy(self.h)
            self.h = None


class Backend:
    """Local compute through a library exporting the C ABI of include/hconv.h."""

    def __init__(self, lib: C.CDLL, device: torch.device, stream_fn=None):
        self.lib = lib
        self.device = device
        self.stream_fn = stream_fn or (lambda: None)

    def _check(self, st):
        _abi.check(self.lib, st)

    def params(self, L, M, m, sym) -> _abi.Params:
        p = _abi.Params()
        self._check(self.lib.hconv_derive_params(L, M, m, sym, C.byref(p)))
        return p

    def block_length(self, p: _abi.Params) -> int:
        return self.lib.hconv_block_length(C.byref(p))

    def forward_lines(self, x: torch.Tensor, p: _abi.Params, r: int, lin: _abi.Lines, F: torch.Tensor,
                      lout: _abi.Lines) -> None:
        self._check(self.lib.hconv_pfft_forward_lines(C.byref(p), C.c_void_p(x.data_ptr()), C.byref(lin), r,
                                                      C.c_void_p(F.data_ptr()), C.byref(lout), self.stream_fn()))

    def backward_lines(self, F: torch.Tensor, p: _abi.Params, r: int, lin: _abi.Lines, h: torch.Tensor,
                       lout: _abi.Lines, accumulate: bool, scale: float) -> None:
        self._check(self.lib.hconv_pfft_backward_lines(C.byref(p), C.c_void_p(F.data_ptr()), C.byref(lin), r,
                                                       C.c_void_p(h.data_ptr()), C.byref(lout), int(accumulate),
                                                       float(scale), self.stream_fn()))

    def plan(self, axes: Sequence[tuple[int, int, int, int]], copies: int, A: int = 2, B: int = 1,
             mult=None) -> _LocalPlan:
        """A plan for `copies` contiguous 1D lines or N-D arrays (product, or `mult`)."""
        d = _abi.Desc()
        d.dims = len(axes)
        for k, (L, M, m, s) in enumerate(axes):
            d.axis[k] = _abi.Axis(L, M, m, s)
        d.A, d.B, d.C, d.dist = A, B, copies, 0
        d.mult = _abi.MULT_PRODUCT if mult is None else mult.kind
        d.device = (self.device.index or 0) if self.device.type == "cuda" else 0
        return _LocalPlan(self, d, None if mult is None or mult.kind == _abi.MULT_PRODUCT else mult)

    def convolve(self, axes: Sequence[tuple[int, int, int, int]], f: torch.Tensor, g: torch.Tensor, copies: int = 1,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """hconv_convolve over contiguous arrays (1D: `copies` rows; N-D: one array)."""
        out = f if out is None else out
        self.plan(axes, copies).convolve([f, g], [out])
        return out


def cuda_backend(device: Optional[torch.device] = None) -> Backend:
    from . import hconv

    dev = device or torch.device("cuda", torch.cuda.current_device())
    return Backend(hconv.lib(), dev, lambda: C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))


def _a2a(recv: torch.Tensor, send: torch.Tensor, rsplit: list[int], ssplit: list[int], group, async_op=False):
    """all_to_all_single on complex data (exchanged as float64 pairs); async_op returns the work
    handle (NCCL: the exchange runs on NCCL's stream, work.wait() orders the current stream)."""
    return dist.all_to_all_single(torch.view_as_real(recv).view(-1), torch.view_as_real(send).view(-1),
                                  [2 * s for s in rsplit], [2 * s for s in ssplit], group=group, async_op=async_op)


@dataclass
class SlabAxis:
    L: int
    M: int
    m: int
    symmetry: int = _abi.COMPLEX


class SlabConvND:
    """x-slab decomposition of a 2D complex or 3D (complex or Hermitian) convolution.

    axes: [x, y] or [x, y, z]; Hermitian mode = z Hermitian (x, y centered).
    Every subtransform size m must be given (tune per axis with hconv.tune_nd beforehand).
    mult: None = builtin product (A = 2, B = 1), else an hconv.MultOperator (A inputs, B outputs).
    """

    def __init__(self, axes: Sequence[SlabAxis], backend: Backend, group=None, mult=None):
        if len(axes) not in (2, 3):
            raise ValueError("slab decomposition is for 2D and 3D convolutions")
        self.axes = list(axes)
        self.b = backend
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.mult = mult
        self.A, self.B = (2, 1) if mult is None else (mult.A, mult.B)
        herm = axes[-1].symmetry == _abi.HERMITIAN
        if len(axes) == 2 and herm:
            raise NotImplementedError("2D Hermitian slabs need the outer axis sharded (3 transposes)")
        self.syms = [(_abi.CENTERED if herm and k < len(axes) - 1 else a.symmetry) for k, a in enumerate(axes)]
        self.data = [((a.L + 1) // 2 if s == _abi.HERMITIAN else a.L) for a, s in zip(axes, self.syms)]
        ay = axes[1]
        self.py = backend.params(ay.L, ay.M, ay.m, self.syms[1])
        self.By = backend.block_length(self.py)
        self.xs = partition(self.data[0], self.G)
        self.ks = partition(self.By, self.G)
        self.inner = self.data[2] if len(axes) == 3 else 1  # z extent (1 for 2D)
        k0, k1 = self.ks[self.rank]
        self.nk = k1 - k0
        x = (axes[0].L, axes[0].M, axes[0].m, self.syms[0])
        sub = [x] if len(axes) == 2 else [x, (axes[2].L, axes[2].M, axes[2].m, self.syms[2])]
        # the (d-1)-D subconvolutions of this rank's nk spectral y-lines: one batched plan
        self.inner_plan = backend.plan(sub, max(1, self.nk), self.A, self.B, mult) if self.nk else None

    def local_shape(self) -> tuple[int, ...]:
        x0, x1 = self.xs[self.rank]
        return (x1 - x0, *self.data[1:])

    def convolve(self, inputs: Sequence[torch.Tensor], out: Optional[Sequence[torch.Tensor]] = None) -> list[torch.Tensor]:
        """inputs: this rank's x-slabs (local_shape()) of the A inputs; returns the B output
        slabs (by default written over the first B inputs)."""
        if isinstance(inputs, torch.Tensor):
            raise TypeError("pass a sequence of input slabs")
        if len(inputs) != self.A:
            raise ValueError(f"expected {self.A} input slabs")
        for t in inputs:
            if tuple(t.shape) != self.local_shape():
                raise ValueError(f"expected local slabs of shape {self.local_shape()}")
        outs = list(inputs[:self.B]) if out is None else list(out)
        if len(outs) != self.B:
            raise ValueError(f"expected {self.B} output slabs")
        G, me, Z, By, nk = self.G, self.rank, self.inner, self.By, self.nk
        nx = inputs[0].shape[0]
        Ly, Lx = self.data[1], self.data[0]
        dev, dt = inputs[0].device, inputs[0].dtype
        nxz = nx * Z
        lin = _lines(nxz, Z, Ly * Z, 1, Z)        # y-lines (x, z) of an x-slab [nx][Ly][Z]
        lspec = _lines(nxz, nxz, 0, 1, nxz)       # the same lines k-major: F[k][x][z]
        send_sizes = [(b - a) * nxz for a, b in self.ks]
        recv_sizes = [nk * (b - a) * Z for a, b in self.xs]
        # one spectral / exchange buffer per input and per output: each exchange runs
        # asynchronously while the next input's forward (or the previous output's backward) computes
        F = [torch.empty(By * nxz, dtype=dt, device=dev) for _ in range(self.A)]
        recv = [torch.empty(sum(recv_sizes), dtype=dt, device=dev) for _ in range(self.A)]
        T = [torch.empty(max(1, nk) * Lx * Z, dtype=dt, device=dev) for _ in range(max(self.A, self.B))]
        back = [torch.empty(sum(recv_sizes), dtype=dt, device=dev) for _ in range(self.B)]
        W = [torch.empty(By * nxz, dtype=dt, device=dev) for _ in range(self.B)]
        # results accumulate in separate buffers when an output aliases an input (inputs are
        # read by every residue's forward)
        ins_ptrs = {t.data_ptr() for t in inputs}
        acc = [torch.empty_like(o) if o.data_ptr() in ins_ptrs else o for o in outs]
        n_res = self.py.n
        scale = 1.0 / (self.py.q * self.py.m)
        for r in range(n_res):
            works = []
            for a in range(self.A):
                self.b.forward_lines(inputs[a], self.py, r, lin, F[a], lspec)
                works.append(_a2a(recv[a], F[a], recv_sizes, send_sizes, self.group, async_op=True))
            for a in range(self.A):
                works[a].wait()
                Ta = T[a].view(max(1, nk), Lx, Z)
                off = 0
                for (xa, xb), sz in zip(self.xs, recv_sizes):
                    if sz:
                        Ta[:, xa:xb, :] = recv[a][off:off + sz].view(nk, xb - xa, Z)
                    off += sz
            if nk:
                self.inner_plan.convolve(T[:self.A], T[:self.B])
            last = r == n_res - 1
            works = []
            for b in range(self.B):
                Tb = T[b].view(max(1, nk), Lx, Z)
                off = 0
                for (xa, xb), sz in zip(self.xs, recv_sizes):
                    if sz:
                        back[b][off:off + sz].view(nk, xb - xa, Z).copy_(Tb[:, xa:xb, :])
                    off += sz
                works.append(_a2a(W[b], back[b], send_sizes, recv_sizes, self.group, async_op=True))
            for b in range(self.B):
                works[b].wait()
                self.b.backward_lines(W[b], self.py, r, lspec, acc[b], lin, accumulate=r > 0,
                                      scale=scale if last else 1.0)
        for o, a_ in zip(outs, acc):
            if o.data_ptr() != a_.data_ptr():
                o.copy_(a_)
        return outs
