"""Host-side mirror of the reference's hybrid-dealiasing interface, backed by the sm_100a
library ``_lib/libhconv_cuda.so`` through the C ABI of ``include/hconv.h``.

Names, argument meaning and error behaviour follow the reference (paths relative to
/root/reference):

* plan module (the reference's only compiled code, proj/include/hconv/plan.hpp:10-108):
  ``Symmetry``, ``Regime``, ``PlanParams``, ``deriveParams``, ``root``, ``RootTable``,
  ``workMemoryWords``, ``name``, ``symmetryFromName``; ``std::invalid_argument`` -> ``ValueError``.
* SPEC modules pfft-complex/-centered/-hermitian: ``forward`` / ``backward``
  (one residue of forward1/2/Inner[C|H] and backward1/2/Inner[C|H], batched).
* SPEC conv1d: ``MultOperator``, ``builtin_mult_product``, ``Conv1dPlan``,
  ``convolve``.
* SPEC convnd: ``AxisSpec``, ``ConvPlanND``, ``convolve_nd``,
  ``hermitian_symmetrize_boundary``.
* SPEC tuner: ``tune_1d`` / ``tune_nd`` -- device-timed (CUDA events).

Data are torch tensors on a CUDA device (complex128; Hermitian residue blocks float64).  There
is no CPU fallback: without the built library or a GPU every call raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import threading
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence, Union

import torch

from . import _abi

import os as _os

# HCONV_LIB_VARIANT=name loads _lib_<name>/libhconv_cuda.so (A/B builds of the same sources with
# different compile-time options, `make VARIANT=name EXTRA=...`); default: the product build
LIB_PATH = _abi.ROOT / ("_lib_" + _os.environ["HCONV_LIB_VARIANT"] if _os.environ.get("HCONV_LIB_VARIANT") else "_lib") \
    / "libhconv_cuda.so"
_lib: Optional[C.CDLL] = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """The CUDA library; raises if it has not been built (no silent fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(f"{LIB_PATH} missing: build it with __graft_entry__.build() (make -C paper_2303_17510_b200)")
            _lib = _abi.bind(C.CDLL(str(LIB_PATH)), ext=True)
        return _lib


def _check(status: int) -> None:
    _abi.check(lib(), status)


class Symmetry(enum.IntEnum):
    """plan.hpp:17 enum class Symmetry."""

    Complex = _abi.COMPLEX
    Centered = _abi.CENTERED
    Hermitian = _abi.HERMITIAN


class Regime(enum.IntEnum):
    """plan.hpp:20 enum class Regime."""

    P1 = _abi.P1
    P2 = _abi.P2
    Inner = _abi.INNER


def name(s: Symmetry) -> str:
    """plan.cpp:10-17."""
    return lib().hconv_symmetry_name(int(s)).decode()


def symmetryFromName(s: str) -> Symmetry:
    """plan.cpp:19-24; unknown names raise ValueError (std::invalid_argument)."""
    out = C.c_int()
    _check(lib().hconv_symmetry_from_name(s.encode(), C.byref(out)))
    return Symmetry(out.value)


@dataclass
class PlanParams:
    """plan.hpp:39-62."""

    L: int = 1
    M: int = 1
    m: int = 1
    p: int = 1
    q: int = 1
    n: int = 1
    D: int = 1
    C: int = 1
    S: int = 1
    inplace: bool = False
    symmetry: Symmetry = Symmetry.Complex
    regime: Regime = Regime.P1

    def _c(self) -> _abi.Params:
        return _abi.Params(self.L, self.M, self.m, self.p, self.q, self.n, self.D, self.C, self.S,
                           int(self.inplace), int(self.symmetry), int(self.regime))

    @classmethod
    def _from_c(cls, p: _abi.Params) -> "PlanParams":
        return cls(p.L, p.M, p.m, p.p, p.q, p.n, p.D, p.C, p.S, bool(p.inplace), Symmetry(p.symmetry), Regime(p.regime))

    def blockLength(self) -> int:  # plan.cpp:26-29
        return lib().hconv_block_length(C.byref(self._c()))

    def residueBlocks(self) -> int:  # plan.hpp:54
        return self.n

    def paddedLength(self) -> int:  # plan.hpp:56
        return self.q * self.m

    def storedLength(self) -> int:  # plan.cpp:31-33
        return lib().hconv_stored_length(C.byref(self._c()))

    def dataLength(self) -> int:
        """Values the kernels read/write per copy (Hermitian: logical 0..ceil(L/2)-1)."""
        return (self.L + 1) // 2 if self.symmetry == Symmetry.Hermitian else self.L


def deriveParams(L: int, M: int, m: int, symmetry: Symmetry = Symmetry.Complex) -> PlanParams:
    """plan.cpp:35-64.  Raises ValueError on L == 0, m == 0 or M < L."""
    out = _abi.Params()
    _check(lib().hconv_derive_params(L, M, m, int(symmetry), C.byref(out)))
    return PlanParams._from_c(out)


def root(N: int, k: int) -> complex:
    """plan.cpp:66-73: zeta_N^k = exp(2 pi i k / N); ValueError for N == 0."""
    re, im = C.c_double(), C.c_double()
    _check(lib().hconv_root(N, k, C.byref(re), C.byref(im)))
    return complex(re.value, im.value)


class RootTable:
    """plan.hpp:84-106: flat table of the N roots zeta_N^k; immutable."""

    def __init__(self, modulus: int):
        buf = (C.c_double * (2 * max(modulus, 1)))()
        _check(lib().hconv_root_table(modulus, C.cast(buf, C.c_void_p)))
        self._N = modulus
        self._z = [complex(buf[2 * k], buf[2 * k + 1]) for k in range(modulus)]

    def modulus(self) -> int:
        return self._N

    def __call__(self, k: int) -> complex:
        return self._z[k % self._N]

    def at(self, a: int, b: int) -> complex:
        return self._z[(a % self._N) * (b % self._N) % self._N]


def workMemoryWords(params: PlanParams, A: int, B: int, d: int, L: int) -> tuple[int, float]:
    """plan.cpp:75-89 -> (implicitWords, explicitWords)."""
    iw, ew = C.c_uint64(), C.c_double()
    _check(lib().hconv_work_memory_words(C.byref(params._c()), A, B, d, L, C.byref(iw), C.byref(ew)))
    return iw.value, ew.value


# ------------------------------------------------------------------------ helpers ----
def _stream(stream) -> C.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _dev(t: torch.Tensor, dtype=torch.complex128) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError("hconv expects CUDA tensors (no CPU fallback)")
    if t.dtype != dtype:
        raise ValueError(f"expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t


# -------------------------------------------------------------- padded FFTs (pfft) ---
def forward(f: torch.Tensor, params: PlanParams, r: int, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """One residue (block) of the padded forward FFT for every row of ``f`` ([C, dataLength]).

    Complex/centered: complex128 [C, blockLength] with F[u m + l] = F_{q l + u n + r}
    (forward1/forward2/forwardInner, forward2C/forwardInnerC).  Hermitian: float64 real
    residues (forward2H/forwardInnerH).  Raises ValueError for r >= n.
    """
    f2 = _dev(f).reshape(-1, f.shape[-1])
    bl = params.blockLength()
    dt = torch.float64 if params.symmetry == Symmetry.Hermitian else torch.complex128
    if out is None:
        out = torch.empty(f2.shape[0], bl, dtype=dt, device=f.device)
    _dev(out, dt)
    p = params._c()
    p.C, p.S = f2.shape[0], 1
    _check(lib().hconv_pfft_forward(C.byref(p), C.c_void_p(f2.data_ptr()), f2.shape[1], r, C.c_void_p(out.data_ptr()), _stream(stream)))
    return out


def forward_conjugate_pair(f: torch.Tensor, params: PlanParams, v: int, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
    """SPEC.md:212-220 forward_conjugate_pair (complex): the residue blocks of v and -v of every
    row of ``f`` from one real/imaginary split, reference order (F_{q l + u n + v}, F_{q l + u n - v}).
    ValueError for a self-paired residue (v == 0 or 2v == n)."""
    f2 = _dev(f).reshape(-1, f.shape[-1])
    bl = params.blockLength()
    Fv = torch.empty(f2.shape[0], bl, dtype=torch.complex128, device=f.device)
    Fn = torch.empty_like(Fv)
    p = params._c()
    p.C, p.S = f2.shape[0], 1
    _check(lib().hconv_pfft_forward_pair(C.byref(p), C.c_void_p(f2.data_ptr()), f2.shape[1], v,
                                         C.c_void_p(Fv.data_ptr()), C.c_void_p(Fn.data_ptr()), _stream(stream)))
    return Fv, Fn


def backward(F: torch.Tensor, params: PlanParams, r: int, h: Optional[torch.Tensor] = None, accumulate: bool = False,
             stream=None) -> torch.Tensor:
    """Unnormalised inverse of one residue (backward1/2/Inner[C|H]); accumulate adds into h."""
    dt = torch.float64 if params.symmetry == Symmetry.Hermitian else torch.complex128
    F2 = _dev(F, dt).reshape(-1, F.shape[-1])
    if h is None:
        h = torch.zeros(F2.shape[0], params.dataLength(), dtype=torch.complex128, device=F.device)
    _dev(h)
    p = params._c()
    p.C, p.S = F2.shape[0], 1
    _check(lib().hconv_pfft_backward(C.byref(p), C.c_void_p(F2.data_ptr()), r, C.c_void_p(h.data_ptr()), h.shape[-1],
                                     int(accumulate), _stream(stream)))
    return h


# ---------------------------------------------------------------- convolutions -------
class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (no copy)."""

    def __init__(self, ptr: int, count: int, real: bool):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8" if real else "<c16",
                                         "data": (ptr, False), "version": 3, "strides": None}


@dataclass(frozen=True)
class MultOperator:
    """SPEC.md:396-399 MultOperator{A, B, apply}: pointwise map of A transformed inputs to B outputs.

    kind MULT_PRODUCT is builtin_mult_product(A) (fused kernels for A = 2).  Otherwise the
    operator is ``apply(blocks, real)``: ``blocks`` are max(A, B) device tensors of one residue
    (complex128, or float64 for a Hermitian innermost axis, whose transformed residues are real,
    PAPER.md:484-485); the A inputs are in blocks[:A] and the B outputs must be left in
    blocks[:B], in place ("F_b <- mult(F_a)").  It runs on the library's stream
    (torch's current stream inside the call).  ``fn`` instead takes the address of a native
    ``hconv_mult_fn`` (include/hconv.h), e.g. a function of the caller's own CUDA library.
    """

    A: int
    B: int
    kind: int = _abi.MULT_PRODUCT
    apply: Optional[Callable] = None
    fn: Optional[int] = None

    def _native(self, host: bool = False):
        """(hconv_mult_fn address, keep-alive object) for the descriptor.  host=True: the
        library passes host pointers (the CPU oracle behind the same ABI, test infrastructure)."""
        if self.kind == _abi.MULT_PRODUCT:
            return None, None
        if self.fn is not None:
            return self.fn, None
        apply = self.apply

        def _fn(F, A, B, count, real, user, stream):
            try:
                if host:
                    import numpy as np

                    n = count * (1 if real else 2)
                    blocks = [torch.from_numpy(np.ctypeslib.as_array(C.cast(F[i], C.POINTER(C.c_double)), (n,))
                                               .view(np.float64 if real else np.complex128))
                              for i in range(max(A, B))]
                    apply(blocks, bool(real))
                    return 0
                dev = torch.cuda.current_device()
                blocks = [torch.as_tensor(_CudaArray(F[i], count, bool(real)), device=f"cuda:{dev}")
                          for i in range(max(A, B))]
                # the library's stream; NULL is the legacy default stream (ExternalStream(0) would
                # be a fresh pool stream, unordered with the library's kernels)
                st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream(dev)
                with torch.cuda.stream(st):
                    apply(blocks, bool(real))
                return 0
            except Exception:  # noqa: BLE001 -- the library turns a nonzero return into a status
                import traceback

                traceback.print_exc()
                return 1

        cb = _abi.MultFn(_fn)
        return C.cast(cb, C.c_void_p).value, cb


def builtin_mult_product(A: int = 2) -> MultOperator:
    """B = 1, elementwise product of the A inputs; ValueError for A < 2."""
    if A < 2:
        raise ValueError("builtin_mult_product requires A >= 2")
    return MultOperator(A, 1, _abi.MULT_PRODUCT)


def mult_operator(A: int, B: int, apply: Callable) -> MultOperator:
    """A general A -> B pointwise operator (see MultOperator)."""
    if A < 1 or B < 1:
        raise ValueError("multiplication operator arity: A >= 1, B >= 1")
    return MultOperator(A, B, _abi.MULT_CALLBACK, apply=apply)


class _Plan:
    def __init__(self, desc: _abi.Desc, mult: "MultOperator"):
        fn, self._keep = mult._native()  # the callback must outlive the plan
        desc.mult_fn = fn
        h = C.c_void_p()
        _check(lib().hconv_plan_create(C.byref(desc), C.byref(h)))
        self._h = h
        self.desc = desc

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hconv_plan_destroy(self._h)
            self._h = None

    def axis_params(self, axis: int) -> PlanParams:
        out = _abi.Params()
        _check(lib().hconv_plan_params(self._h, axis, C.byref(out)))
        return PlanParams._from_c(out)

    def kernel(self, axis: int = 0) -> str:
        return lib().hconv_plan_kernel(self._h, axis).decode()

    def planner_report(self) -> tuple[list[dict], bool]:
        W = 7  # hconv_ext.h: (m, p, q, n, block, median ms, explicit) per row
        buf = (C.c_double * (W * 256))()
        k = lib().hconv_plan_report(self._h, buf, 256)
        cached = k < 0
        k = -k - 1 if cached else k
        rows = [dict(m=int(buf[W * i]), p=int(buf[W * i + 1]), q=int(buf[W * i + 2]), n=int(buf[W * i + 3]),
                     block=int(buf[W * i + 4]), median_ms=buf[W * i + 5], explicit=bool(buf[W * i + 6]))
                for i in range(k)]
        return rows, cached

    def workspace_bytes(self) -> int:
        return lib().hconv_plan_workspace_bytes(self._h)

    def _run(self, inputs: Sequence[torch.Tensor], outs: Sequence[torch.Tensor], stream) -> None:
        ins = (C.c_void_p * len(inputs))(*[t.data_ptr() for t in inputs])
        o = (C.c_void_p * len(outs))(*[t.data_ptr() for t in outs])
        _check(lib().hconv_convolve(self._h, ins, o, _stream(stream)))

    def _run_host(self, inputs: Sequence[torch.Tensor], outs: Sequence[torch.Tensor]) -> None:
        ins = (C.c_void_p * len(inputs))(*[t.data_ptr() for t in inputs])
        o = (C.c_void_p * len(outs))(*[t.data_ptr() for t in outs])
        _check(lib().hconv_convolve_host(self._h, ins, o))


class Conv1dPlan(_Plan):
    """1D dealiased convolution of C copies ([C, dist] complex128 rows).

    m=None runs the device-timed planner (tune_1d) over the 7-smooth sizes whose block length
    has a kernel; the chosen (m, p, q, n) is in ``params``.
    """

    def __init__(self, L: int, M: int, m: Optional[int] = None, symmetry: Symmetry = Symmetry.Complex,
                 mult: Optional[MultOperator] = None, C_: int = 1, dist: int = 0, device: int = 0):
        mult = mult or builtin_mult_product(2)
        d = _abi.Desc()
        d.dims = 1
        d.axis[0] = _abi.Axis(L, M, m or 0, int(symmetry))
        d.A, d.B, d.mult, d.C, d.dist, d.device = mult.A, mult.B, mult.kind, C_, dist, device
        super().__init__(d, mult)
        self.mult = mult
        self.params = self.axis_params(0)


@dataclass
class AxisSpec:
    """SPEC.md:465-468 (stride/copies are implied by the contiguous [x][y][z] layout)."""

    L: int
    M: int
    m: Optional[int] = None
    symmetry: Symmetry = Symmetry.Complex


FLAG_MIN_MEMORY = 1  # include/hconv.h HCONV_FLAG_MIN_MEMORY


class ConvPlanND(_Plan):
    """d-dimensional plan; axes[-1] is the contiguous innermost axis.
    Hermitian mode (innermost Hermitian) makes the outer axes centered."""

    def __init__(self, axes: Sequence[AxisSpec], mult: Optional[MultOperator] = None, device: int = 0, C_: int = 1,
                 min_memory: bool = False):
        """min_memory: reuse one subconvolution work buffer per outer plane (HCONV_FLAG_MIN_MEMORY,
        the paper's (A+B) p m L^{d-1} work bound) instead of batching every plane."""
        mult = mult or builtin_mult_product(2)
        if not 1 <= len(axes) <= 3:
            raise ValueError("1 to 3 axes")
        d = _abi.Desc()
        d.dims = len(axes)
        for k, a in enumerate(axes):
            d.axis[k] = _abi.Axis(a.L, a.M, a.m or 0, int(a.symmetry))
        d.A, d.B, d.mult, d.C, d.dist, d.device = mult.A, mult.B, mult.kind, C_, 0, device
        d.flags = FLAG_MIN_MEMORY if min_memory else 0
        super().__init__(d, mult)
        self.copies = C_
        self.mult = mult
        self.axes = list(axes)
        self.params = [self.axis_params(k) for k in range(len(axes))]

    def shape(self) -> tuple[int, ...]:
        """array shape a call expects: (C, *axes) for a batch of C > 1 arrays"""
        shp = tuple(p.dataLength() for p in self.params)
        return (self.copies, *shp) if self.copies > 1 else shp


def _check_mult(inputs, mult: MultOperator, plan: _Plan):
    if len(inputs) != mult.A or mult.A != plan.desc.A or mult.B != plan.desc.B:
        raise ValueError("arity mismatch between inputs, mult and plan (SPEC.md:410)")


Outs = Optional[Union[torch.Tensor, Sequence[torch.Tensor]]]


def _outs(out: Outs, ins: Sequence[torch.Tensor], B: int, conv) -> list[torch.Tensor]:
    """B output arrays: by default the first B inputs (overwritten in place)."""
    if out is None:
        if B > len(ins):
            raise ValueError("B > A: pass the B output arrays explicitly")
        return list(ins[:B])
    outs = [out] if isinstance(out, torch.Tensor) else list(out)
    if len(outs) != B:
        raise ValueError(f"expected {B} output arrays")
    return [conv(o) for o in outs]


def convolve(inputs: Sequence[torch.Tensor], mult: MultOperator, plan: Conv1dPlan, out: Outs = None,
             stream=None) -> list[torch.Tensor]:
    """Alg. convolve / convolveX: returns the B outputs [h_0 .. h_{B-1}]; by
    default they overwrite the first B inputs (the reference's in-place convention)."""
    _check_mult(inputs, mult, plan)
    ins = [_dev(t) for t in inputs]
    rows = plan.desc.C
    need = (rows - 1) * (plan.desc.dist or plan.params.dataLength()) + plan.params.dataLength()
    outs = _outs(out, ins, mult.B, _dev)
    for t in ins + outs:
        if t.numel() < need:
            raise ValueError("array smaller than the plan's C x dist layout")
    plan._run(ins, outs, stream)
    return outs


def convolve_nd(inputs: Sequence[torch.Tensor], mult: MultOperator, plan: ConvPlanND, out: Outs = None,
                stream=None) -> list[torch.Tensor]:
    """convolve_nd over contiguous arrays of shape plan.shape()."""
    _check_mult(inputs, mult, plan)
    shp = plan.shape()
    ins = [_dev(t) for t in inputs]
    outs = _outs(out, ins, mult.B, _dev)
    for t in ins + outs:
        if tuple(t.shape) != shp:
            raise ValueError(f"expected shape {shp}, got {tuple(t.shape)}")
    plan._run(ins, outs, stream)
    return outs


def _host(t: torch.Tensor) -> torch.Tensor:
    if t.is_cuda or t.dtype != torch.complex128 or not t.is_contiguous():
        raise ValueError("convolve_host expects contiguous complex128 CPU tensors")
    return t


def convolve_host(inputs: Sequence[torch.Tensor], mult: MultOperator, plan: "_Plan",
                  out: Outs = None) -> list[torch.Tensor]:
    """convolve / convolve_nd on HOST tensors -- the reference library's calling convention
    (synchronous, host arrays).  The library streams a 1D batch through the device in chunks,
    overlapping host->device copies, the convolution and device->host copies (pin the tensors,
    ``t.pin_memory()``, for the overlap).  Computes on the GPU; there is no CPU path."""
    _check_mult(inputs, mult, plan)
    ins = [_host(t) for t in inputs]
    outs = _outs(out, ins, mult.B, _host)
    if isinstance(plan, ConvPlanND):
        shp = plan.shape()
        for t in ins + outs:
            if tuple(t.shape) != shp:
                raise ValueError(f"expected shape {shp}, got {tuple(t.shape)}")
    else:
        need = (plan.desc.C - 1) * (plan.desc.dist or plan.params.dataLength()) + plan.params.dataLength()
        for t in ins + outs:
            if t.numel() < need:
                raise ValueError("array smaller than the plan's C x dist layout")
    plan._run_host(ins, outs)
    return outs


def hermitian_symmetrize_boundary(f: torch.Tensor, Ls: Sequence[int]) -> torch.Tensor:
    """enforce f(-x,-y,0) = conj f(x,y,0) on the innermost-index-0 hyperplane
    of a centered/.../Hermitian array (outer axes centered, origin at floor(L/2)); in place."""
    plane = f[..., 0]
    outer = list(Ls[:-1])
    idx = [torch.arange(L, device=f.device) for L in outer]
    # mirrored index of stored i along a centered axis: -(i - H) + H = 2H - i (invalid if >= L)
    mirror = [2 * (L // 2) - ix for L, ix in zip(outer, idx)]
    grids = torch.meshgrid(*idx, indexing="ij")
    mgrids = torch.meshgrid(*mirror, indexing="ij")
    valid = torch.ones_like(grids[0], dtype=torch.bool)
    for L, mg in zip(outer, mgrids):
        valid &= (mg >= 0) & (mg < L)
    # lexicographic "negative half": first nonzero logical coordinate (last axis first) < 0
    neg = torch.zeros_like(valid)
    decided = torch.zeros_like(valid)
    for L, g in reversed(list(zip(outer, grids))):
        c = g - L // 2
        neg |= (~decided) & (c < 0)
        decided |= c != 0
    src = plane.clone()
    mg_clamped = [mg.clamp(0, L - 1) for L, mg in zip(outer, mgrids)]
    mirrored = src[tuple(mg_clamped)].conj()
    new = torch.where(neg, mirrored, src)
    new = torch.where(valid, new, torch.zeros_like(new))
    origin = tuple(L // 2 for L in outer)
    new[origin] = new[origin].real.to(new.dtype)
    plane.copy_(new)
    return f


# ------------------------------------------------------------------------ tuner ------
def tune_1d(L: int, M: int, symmetry: Symmetry = Symmetry.Complex, C_: int = 1, mult: Optional[MultOperator] = None,
            device: int = 0) -> tuple[PlanParams, list[dict], bool]:
    """SPEC.md:533-541 on the device: returns (chosen params, timed candidates, cached)."""
    plan = Conv1dPlan(L, M, None, symmetry, mult, C_, 0, device)
    rows, cached = plan.planner_report()
    return plan.params, rows, cached


def tune_nd(axes: Sequence[AxisSpec], mult: Optional[MultOperator] = None, device: int = 0) -> ConvPlanND:
    """each axis tuned independently."""
    return ConvPlanND([AxisSpec(a.L, a.M, None, a.symmetry) for a in axes], mult, device)


class CapturedConvolution:
    """A convolution captured once into a CUDA graph and replayed: the kernels of
    convolve / convolve_nd on fixed device arrays without the host-side launch path (Python,
    ctypes, plan bookkeeping) between steps -- what bounds small problems (config 1: 1024 lines
    of 1024 points take ~40 us on the device, about as long as issuing the call).  The plan's
    work buffers are allocated by the warm-up call before capture.  Built-in product or native
    (fn=) operators only: a Python operator cannot be captured."""

    def __init__(self, inputs: Sequence[torch.Tensor], mult: MultOperator, plan: "_Plan", out: Outs = None):
        if mult.kind != _abi.MULT_PRODUCT and mult.apply is not None:
            raise ValueError("a Python multiplication operator cannot be captured in a CUDA graph")
        if out is None:
            raise ValueError("CapturedConvolution needs explicit output arrays: in place, the warm-up "
                             "call would overwrite the inputs and every replay would convolve its own output")
        outs_ = [out] if isinstance(out, torch.Tensor) else list(out)
        for o in outs_:
            for t in inputs:
                if o.untyped_storage().data_ptr() == t.untyped_storage().data_ptr():
                    raise ValueError("CapturedConvolution: an output array aliases an input array")
        run = convolve_nd if isinstance(plan, ConvPlanND) else convolve
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.outs = run(inputs, mult, plan, out)  # warm-up: allocates the plan's scratch
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            run(inputs, mult, plan, self.outs)
        self._keep = (list(inputs), plan)

    def __call__(self) -> list[torch.Tensor]:
        self.graph.replay()
        return self.outs


def fill_uniform(t: torch.Tensor, seed: int, a: int, first_index: int = 0, stream=None) -> torch.Tensor:
    """Counter-based synthetic inputs written on the device."""
    _dev(t)
    _check(lib().hconv_util_fill_uniform(seed, a, first_index, t.numel(), C.c_void_p(t.data_ptr()), _stream(stream)))
    return t
