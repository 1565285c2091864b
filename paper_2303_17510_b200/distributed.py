"""Slab-decomposed 2D/3D dealiased convolution over several GPUs.

The reference has no distributed code (SPEC.md:512 lists MPI decomposition as a non-goal); this
is the multi-GPU extension the north star asks for, built on the same C ABI.

Layout: the contiguous arrays [x][y] (2D) or [x][y][z] (3D, z innermost) are split into x-slabs,
rank g owning rows [x0_g, x1_g).  Because a padded FFT needs its whole axis, the OUTER padded
transform runs along y, which every rank holds completely; the sharded axis x becomes an inner
axis after one all-to-all transpose:

  for each residue block r of the y axis (PAPER.md:584-600 with y as the outer axis):
    1. local forward padded y-FFT of the A inputs        (hconv_pfft_forward, block r)
    2. all-to-all: rank g receives the spectral y-lines of its block [k0_g, k1_g) for ALL x
    3. local (d-1)-D subconvolutions over (x[, z]) of those lines (hconv_convolve; owns mult)
    4. all-to-all back to the x-slab owners
    5. local inverse padded y-FFT of block r, accumulated          (hconv_pfft_backward)
  h *= 1 / (q_y m_y)

The multi-D DFT is separable, so this equals the paper's x-outer recursion numerically.  Exactly
two exchanges per residue carry (A + B) x L_x x B_y x (inner) values.  The collective is
torch.distributed all_to_all_single (NCCL over NVLink on GPUs; gloo on CPU in the tests).

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

    def forward(self, x: torch.Tensor, p: _abi.Params, r: int, copies: int, stride: int, dist_: int) -> torch.Tensor:
        """Residue r of the padded forward FFT of `copies` lines (element stride `stride`,
        copy distance `dist_`) of the contiguous complex128 tensor x -> [copies, blockLength]."""
        q = _abi.Params.from_buffer_copy(p)
        q.C, q.S = copies, stride
        out = torch.empty(copies, self.block_length(p), dtype=torch.complex128, device=self.device)
        self._check(self.lib.hconv_pfft_forward(C.byref(q), C.c_void_p(x.data_ptr()), dist_, r,
                                                C.c_void_p(out.data_ptr()), self.stream_fn()))
        return out

    def backward(self, F: torch.Tensor, p: _abi.Params, r: int, h: torch.Tensor, copies: int, stride: int, dist_: int,
                 accumulate: bool) -> None:
        q = _abi.Params.from_buffer_copy(p)
        q.C, q.S = copies, stride
        self._check(self.lib.hconv_pfft_backward(C.byref(q), C.c_void_p(F.data_ptr()), r, C.c_void_p(h.data_ptr()),
                                                 dist_, int(accumulate), self.stream_fn()))

    def convolve(self, axes: Sequence[tuple[int, int, int, int]], f: torch.Tensor, g: torch.Tensor, copies: int = 1,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """hconv_convolve over contiguous arrays (1D: `copies` rows; N-D: one array)."""
        d = _abi.Desc()
        d.dims = len(axes)
        for k, (L, M, m, s) in enumerate(axes):
            d.axis[k] = _abi.Axis(L, M, m, s)
        d.A, d.B, d.mult, d.C, d.dist = 2, 1, _abi.MULT_PRODUCT, copies, 0
        d.device = self.device.index or 0 if self.device.type == "cuda" else 0
        h = C.c_void_p()
        self._check(self.lib.hconv_plan_create(C.byref(d), C.byref(h)))
        out = f if out is None else out
        try:
            ins = (C.c_void_p * 2)(f.data_ptr(), g.data_ptr())
            outs = (C.c_void_p * 1)(out.data_ptr())
            self._check(self.lib.hconv_convolve(h, ins, outs, self.stream_fn()))
        finally:
            self.lib.hconv_plan_destroy(h)
        return out


def cuda_backend(device: Optional[torch.device] = None) -> Backend:
    from . import hconv

    dev = device or torch.device("cuda", torch.cuda.current_device())
    return Backend(hconv.lib(), dev, lambda: C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))


def _a2a(recv: torch.Tensor, send: torch.Tensor, rsplit: list[int], ssplit: list[int], group) -> None:
    """all_to_all_single on complex data (exchanged as float64 pairs)."""
    dist.all_to_all_single(torch.view_as_real(recv).view(-1), torch.view_as_real(send).view(-1),
                           [2 * s for s in rsplit], [2 * s for s in ssplit], group=group)


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
    """

    def __init__(self, axes: Sequence[SlabAxis], backend: Backend, group=None):
        if len(axes) not in (2, 3):
            raise ValueError("slab decomposition is for 2D and 3D convolutions")
        self.axes = list(axes)
        self.b = backend
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
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

    def local_shape(self) -> tuple[int, ...]:
        x0, x1 = self.xs[self.rank]
        return (x1 - x0, *self.data[1:])

    def _forward_y(self, f: torch.Tensor, r: int) -> torch.Tensor:
        """[nx, Ly, Z] -> [nx, Z, By] (residue r of the y padded FFT)."""
        nx, Z = f.shape[0], self.inner
        Ly = self.data[1]
        if Z == 1:
            return self.b.forward(f, self.py, r, nx, 1, Ly).view(nx, 1, self.By)
        out = torch.empty(nx, Z, self.By, dtype=f.dtype, device=f.device)
        for i in range(nx):
            out[i] = self.b.forward(f[i], self.py, r, Z, Z, 1)
        return out

    def _backward_y(self, W: torch.Tensor, r: int, h: torch.Tensor, accumulate: bool) -> None:
        nx, Z = W.shape[0], self.inner
        Ly = self.data[1]
        if Z == 1:
            self.b.backward(W.reshape(nx, self.By).contiguous(), self.py, r, h, nx, 1, Ly, accumulate)
            return
        for i in range(nx):
            self.b.backward(W[i].contiguous(), self.py, r, h[i], Z, Z, 1, accumulate)

    def _inner(self, T: torch.Tensor, U: torch.Tensor) -> None:
        """(d-1)-D subconvolutions of the received spectral lines T, U: [nk, Lx, Z], in place in T."""
        ax = self.axes
        x = (ax[0].L, ax[0].M, ax[0].m, self.syms[0])
        if self.inner == 1:
            self.b.convolve([x], T.view(T.shape[0], -1), U.view(U.shape[0], -1), copies=T.shape[0])
        else:
            z = (ax[2].L, ax[2].M, ax[2].m, self.syms[2])
            for k in range(T.shape[0]):
                self.b.convolve([x, z], T[k], U[k])

    def convolve(self, f: torch.Tensor, g: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """f, g: this rank's x-slabs (local_shape()); returns the convolution's x-slab."""
        if tuple(f.shape) != self.local_shape() or tuple(g.shape) != self.local_shape():
            raise ValueError(f"expected local slabs of shape {self.local_shape()}")
        G, me = self.G, self.rank
        nx = f.shape[0]
        Z = self.inner
        f3, g3 = f.reshape(nx, self.data[1], Z), g.reshape(nx, self.data[1], Z)
        h = torch.zeros_like(f3) if out is None else out.reshape(nx, self.data[1], Z)
        k0, k1 = self.ks[me]
        nk = k1 - k0
        Lx = self.data[0]
        send_sizes = [nx * Z * (b - a) for a, b in self.ks]
        recv_sizes = [(b - a) * Z * nk for a, b in self.xs]
        n_res = self.py.n
        for r in range(n_res):
            specs = []
            for a in (f3, g3):
                F = self._forward_y(a, r)  # [nx, Z, By]
                send = torch.cat([F[:, :, a_:b_].permute(2, 0, 1).reshape(-1) for a_, b_ in self.ks])
                recv = torch.empty(sum(recv_sizes), dtype=F.dtype, device=F.device)
                _a2a(recv, send, recv_sizes, send_sizes, self.group)
                # pieces from rank h: [nk, nx_h, Z] -> T[nk, Lx, Z]
                T = torch.empty(nk, Lx, Z, dtype=F.dtype, device=F.device)
                off = 0
                for (xa, xb), sz in zip(self.xs, recv_sizes):
                    T[:, xa:xb, :] = recv[off:off + sz].view(nk, xb - xa, Z)
                    off += sz
                specs.append(T)
            self._inner(specs[0], specs[1])
            T = specs[0]
            send = torch.cat([T[:, xa:xb, :].reshape(-1) for xa, xb in self.xs])
            back = torch.empty(sum(send_sizes), dtype=T.dtype, device=T.device)
            _a2a(back, send, send_sizes, recv_sizes, self.group)
            W = torch.empty(nx, Z, self.By, dtype=T.dtype, device=T.device)
            off = 0
            for (a_, b_), sz in zip(self.ks, send_sizes):
                W[:, :, a_:b_] = back[off:off + sz].view(b_ - a_, nx, Z).permute(1, 2, 0)
                off += sz
            self._backward_y(W, r, h, accumulate=r > 0)
        h.mul_(1.0 / (self.py.q * self.py.m))
        return h.reshape(self.local_shape())
