"""Test-side loader of the CPU oracle (oracle/_build/libhconv_oracle.so) and of the reference's
own plan module compiled from /root/reference (oracle/_ref/libplanref.so).  TEST
INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's CPU arm use it."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_2303_17510_b200 import _abi

REPO = Path(__file__).resolve().parents[1]
ORACLE = REPO / "oracle" / "_build" / "libhconv_oracle.so"
REF = REPO / "oracle" / "_ref" / "libplanref.so"

_dp = C.POINTER(C.c_double)


def _build():
    if not ORACLE.exists():
        subprocess.run(["make", "-C", str(REPO / "oracle")], check=True, capture_output=True)


def load() -> C.CDLL:
    _build()
    lib = _abi.bind(C.CDLL(str(ORACLE)))
    P = C.POINTER(_abi.Params)
    for name, args in {
        "oracle_naive_dft": [_dp, C.c_size_t, C.c_int, _dp],
        "oracle_fft": [_dp, C.c_size_t, C.c_int, _dp],
        "oracle_padded_dft_slice": [P, _dp, C.c_size_t, _dp],
        "oracle_forward": [P, _dp, C.c_size_t, _dp],
        "oracle_backward": [P, _dp, C.c_size_t, _dp],
        "oracle_forward_conjugate_pair": [P, _dp, C.c_size_t, _dp, _dp],
        "oracle_direct_convolution": [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_size_t), _dp, _dp, _dp],
        "oracle_symmetrize_boundary": [C.c_int, C.POINTER(C.c_size_t), _dp],
        "oracle_set_threads": [C.c_int],
    }.items():
        fn = getattr(lib, name)
        fn.restype = C.c_int
        fn.argtypes = args
    lib.oracle_fill_uniform.restype = None
    lib.oracle_fill_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_size_t, _dp]
    return lib


def load_ref() -> C.CDLL | None:
    if not REF.exists():
        return None
    lib = C.CDLL(str(REF))
    lib.ref_derive_params.argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.POINTER(C.c_uint64)]
    lib.ref_lengths.argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.POINTER(C.c_uint64)]
    lib.ref_root.argtypes = [C.c_size_t, C.c_int64, _dp, _dp]
    lib.ref_work_memory_words.argtypes = [C.c_size_t] * 3 + [C.c_int] + [C.c_size_t] * 4 + [C.POINTER(C.c_uint64), _dp]
    lib.ref_root_table.argtypes = [C.c_size_t, C.c_int64, C.c_size_t, _dp]
    lib.ref_root_table_at.argtypes = [C.c_size_t, C.c_uint64, C.c_uint64, _dp, _dp]
    lib.ref_symmetry_name.restype = C.c_char_p
    lib.ref_symmetry_from_name.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
    return lib


def ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class Oracle:
    """Thin numpy-facing wrapper around the oracle library."""

    def __init__(self):
        self.lib = load()

    def derive(self, L, M, m, sym=0) -> _abi.Params:
        p = _abi.Params()
        _abi.check(self.lib, self.lib.hconv_derive_params(L, M, m, sym, C.byref(p)))
        return p

    def block_length(self, p) -> int:
        return self.lib.hconv_block_length(C.byref(p))

    @staticmethod
    def data_length(p) -> int:
        return (p.L + 1) // 2 if p.symmetry == _abi.HERMITIAN else p.L

    def forward(self, p, f: np.ndarray, r: int) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.complex128)
        F = np.zeros(self.block_length(p), np.complex128)
        assert self.lib.oracle_forward(C.byref(p), ptr(f.view(np.float64)), r, ptr(F.view(np.float64))) == 0
        return F.real.copy() if p.symmetry == _abi.HERMITIAN else F

    def backward(self, p, F: np.ndarray, r: int) -> np.ndarray:
        Fc = np.ascontiguousarray(F, dtype=np.complex128)
        V = np.zeros(self.data_length(p), np.complex128)
        assert self.lib.oracle_backward(C.byref(p), ptr(Fc.view(np.float64)), r, ptr(V.view(np.float64))) == 0
        return V

    def slice(self, p, f: np.ndarray, r: int) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.complex128)
        F = np.zeros(self.block_length(p), np.complex128)
        assert self.lib.oracle_padded_dft_slice(C.byref(p), ptr(f.view(np.float64)), r, ptr(F.view(np.float64))) == 0
        return F.real.copy() if p.symmetry == _abi.HERMITIAN else F

    def conjugate_pair(self, p, f, v):
        f = np.ascontiguousarray(f, dtype=np.complex128)
        a = np.zeros(self.block_length(p), np.complex128)
        b = np.zeros_like(a)
        assert self.lib.oracle_forward_conjugate_pair(C.byref(p), ptr(f.view(np.float64)), v, ptr(a.view(np.float64)),
                                                      ptr(b.view(np.float64))) == 0
        return a, b

    def dft(self, x, sign=1, naive=True):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.zeros_like(x)
        fn = self.lib.oracle_naive_dft if naive else self.lib.oracle_fft
        assert fn(ptr(x.view(np.float64)), x.size, sign, ptr(y.view(np.float64))) == 0
        return y

    def convolve(self, axes, f, g, C_=1, dist=0):
        """axes: list of (L, M, m, sym); f, g contiguous complex128 arrays."""
        d = _abi.Desc()
        d.dims = len(axes)
        for k, (L, M, m, s) in enumerate(axes):
            d.axis[k] = _abi.Axis(L, M, m, s)
        d.A, d.B, d.mult, d.C, d.dist = 2, 1, 0, C_, dist
        h = C.c_void_p()
        _abi.check(self.lib, self.lib.hconv_plan_create(C.byref(d), C.byref(h)))
        f = np.ascontiguousarray(f, dtype=np.complex128)
        g = np.ascontiguousarray(g, dtype=np.complex128)
        out = np.zeros_like(f)
        ins = (C.c_void_p * 2)(f.ctypes.data, g.ctypes.data)
        outs = (C.c_void_p * 1)(out.ctypes.data)
        try:
            _abi.check(self.lib, self.lib.hconv_convolve(h, ins, outs, None))
        finally:
            self.lib.hconv_plan_destroy(h)
        return out

    def convolve_general(self, axes, inputs, B=1, apply=None, C_=1, dist=0):
        """hconv_convolve with A = len(inputs) inputs and B outputs.  apply=None: builtin
        product (B must be 1); else apply(blocks, real) is the operator on numpy views of the
        max(A, B) transformed blocks (complex128, or float64 when real), in place."""
        A = len(inputs)
        d = _abi.Desc()
        d.dims = len(axes)
        for k, (L, M, m, s) in enumerate(axes):
            d.axis[k] = _abi.Axis(L, M, m, s)
        d.A, d.B, d.C, d.dist = A, B, C_, dist
        cb = None
        if apply is None:
            d.mult = _abi.MULT_PRODUCT
        else:
            def _fn(F, A_, B_, count, real, user, stream):
                try:
                    dt = np.float64 if real else np.complex128
                    blocks = [np.ctypeslib.as_array(C.cast(F[i], C.POINTER(C.c_double)), (count * (1 if real else 2),)).view(dt)
                              for i in range(max(A_, B_))]
                    apply(blocks, bool(real))
                    return 0
                except Exception:  # noqa: BLE001 -- reported as a status by the library
                    return 1
            cb = _abi.MultFn(_fn)
            d.mult = _abi.MULT_CALLBACK
            d.mult_fn = C.cast(cb, C.c_void_p)
        h = C.c_void_p()
        _abi.check(self.lib, self.lib.hconv_plan_create(C.byref(d), C.byref(h)))
        ins = [np.ascontiguousarray(x, dtype=np.complex128) for x in inputs]
        outs = [np.zeros_like(ins[0]) for _ in range(B)]
        try:
            _abi.check(self.lib, self.lib.hconv_convolve(h, (C.c_void_p * A)(*[x.ctypes.data for x in ins]),
                                                         (C.c_void_p * B)(*[o.ctypes.data for o in outs]), None))
        finally:
            self.lib.hconv_plan_destroy(h)
        return outs

    def direct(self, syms, Ls, f, g):
        f = np.ascontiguousarray(f, dtype=np.complex128)
        g = np.ascontiguousarray(g, dtype=np.complex128)
        out = np.zeros_like(f)
        S = (C.c_int * len(syms))(*syms)
        LL = (C.c_size_t * len(Ls))(*Ls)
        assert self.lib.oracle_direct_convolution(len(syms), S, LL, ptr(f.view(np.float64)), ptr(g.view(np.float64)),
                                                  ptr(out.view(np.float64))) == 0
        return out

    def symmetrize(self, Ls, f):
        f = np.ascontiguousarray(f, dtype=np.complex128)
        LL = (C.c_size_t * len(Ls))(*Ls)
        assert self.lib.oracle_symmetrize_boundary(len(Ls), LL, ptr(f.view(np.float64))) == 0
        return f

    def uniform(self, seed, a, count, first=0):
        out = np.zeros(count, np.complex128)
        self.lib.oracle_fill_uniform(seed, a, first, count, ptr(out.view(np.float64)))
        return out


def rel_l2(x, ref) -> float:
    x = np.asarray(x)
    ref = np.asarray(ref)
    den = np.linalg.norm(ref.ravel())
    return float(np.linalg.norm((x - ref).ravel()) / (den if den > 0 else 1.0))
