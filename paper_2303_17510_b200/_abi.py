"""ctypes view of the C ABI declared in include/hconv.h (structs, status codes, prototypes).

Shared by every library that exports the ABI; this module only describes the boundary and
never chooses which library implements it.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

ROOT = Path(__file__).resolve().parent
REPO = ROOT.parent

OK, INVALID_ARG, UNSUPPORTED, CUDA_ERROR, NCCL_ERROR, ALLOC, INTERNAL = range(7)
COMPLEX, CENTERED, HERMITIAN = 0, 1, 2
P1, P2, INNER = 0, 1, 2
MULT_PRODUCT, MULT_CALLBACK = 0, 1

# include/hconv.h hconv_mult_fn: (F, A, B, count, real, user, stream) -> int (0 = success)
MultFn = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_void_p), C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.c_void_p,
                     C.c_void_p)


# include/hconv.h hconv_exchange_fn: (send, scounts, sdispls, recv, rcounts, rdispls, user, stream) -> int
ExchangeFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.c_void_p,
                         C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.c_void_p, C.c_void_p)


class Slab(C.Structure):
    """hconv_slab: x-slab decomposition over `nranks` ranks (NCCL communicator or callback)."""

    _fields_ = [
        ("rank", C.c_int),
        ("nranks", C.c_int),
        ("nccl_comm", C.c_void_p),
        ("exchange", C.c_void_p),
        ("exchange_user", C.c_void_p),
        ("chunks", C.c_size_t),
    ]


class Params(C.Structure):
    """hconv_params == proj/include/hconv/plan.hpp:39-62 PlanParams."""

    _fields_ = [(n, C.c_size_t) for n in "L M m p q n D C S".split()] + [
        ("inplace", C.c_int),
        ("symmetry", C.c_int),
        ("regime", C.c_int),
    ]


class Axis(C.Structure):
    _fields_ = [("L", C.c_size_t), ("M", C.c_size_t), ("m", C.c_size_t), ("symmetry", C.c_int)]


class Desc(C.Structure):
    _fields_ = [
        ("dims", C.c_int),
        ("axis", Axis * 3),
        ("A", C.c_size_t),
        ("B", C.c_size_t),
        ("mult", C.c_int),
        ("C", C.c_size_t),
        ("dist", C.c_size_t),
        ("device", C.c_int),
        ("flags", C.c_int),
        ("mult_fn", C.c_void_p),
        ("mult_user", C.c_void_p),
        ("slab", C.c_void_p),
    ]


class Lines(C.Structure):
    """hconv_lines: line l starts at (l // nin) * d_out + (l % nin) * d_in, values at stride es."""

    _fields_ = [(n, C.c_size_t) for n in ("count", "nin", "d_out", "d_in", "es")]


# symbol -> (restype, argtypes); every symbol include/hconv.h declares
PROTOTYPES = {
    "hconv_derive_params": (C.c_int, [C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.POINTER(Params)]),
    "hconv_block_length": (C.c_size_t, [C.POINTER(Params)]),
    "hconv_stored_length": (C.c_size_t, [C.POINTER(Params)]),
    "hconv_padded_length": (C.c_size_t, [C.POINTER(Params)]),
    "hconv_root": (C.c_int, [C.c_size_t, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "hconv_work_memory_words": (
        C.c_int,
        [C.POINTER(Params), C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.POINTER(C.c_uint64), C.POINTER(C.c_double)],
    ),
    "hconv_root_table": (C.c_int, [C.c_size_t, C.c_void_p]),
    "hconv_symmetry_name": (C.c_char_p, [C.c_int]),
    "hconv_symmetry_from_name": (C.c_int, [C.c_char_p, C.POINTER(C.c_int)]),
    "hconv_pfft_forward": (C.c_int, [C.POINTER(Params), C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p, C.c_void_p]),
    "hconv_pfft_backward": (
        C.c_int,
        [C.POINTER(Params), C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p],
    ),
    "hconv_pfft_forward_pair": (
        C.c_int, [C.POINTER(Params), C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p],
    ),
    "hconv_pfft_forward_lines": (
        C.c_int,
        [C.POINTER(Params), C.c_void_p, C.POINTER(Lines), C.c_size_t, C.c_void_p, C.POINTER(Lines), C.c_void_p],
    ),
    "hconv_pfft_backward_lines": (
        C.c_int,
        [C.POINTER(Params), C.c_void_p, C.POINTER(Lines), C.c_size_t, C.c_void_p, C.POINTER(Lines), C.c_int, C.c_double,
         C.c_void_p],
    ),
    "hconv_plan_create": (C.c_int, [C.POINTER(Desc), C.POINTER(C.c_void_p)]),
    "hconv_plan_params": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(Params)]),
    "hconv_plan_slab": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "hconv_plan_workspace_bytes": (C.c_size_t, [C.c_void_p]),
    "hconv_convolve": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_void_p]),
    "hconv_convolve_host": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "hconv_plan_destroy": (C.c_int, [C.c_void_p]),
    "hconv_last_error": (C.c_char_p, []),
    "hconv_backend": (C.c_char_p, []),
}

# include/hconv_ext.h (CUDA library only)
EXT_PROTOTYPES = {
    "hconv_util_fill_uniform": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_size_t, C.c_void_p, C.c_void_p]),
    "hconv_plan_report": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_int]),
    "hconv_plan_kernel": (C.c_char_p, [C.c_void_p, C.c_int]),
    "hconv_example_mult": (C.c_void_p, [C.c_int]),
    "hconv_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "hconv_nccl_comm_init": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "hconv_nccl_comm_destroy": (C.c_int, [C.c_void_p]),
}


def bind(lib: C.CDLL, ext: bool = False) -> C.CDLL:
    for name, (res, args) in {**PROTOTYPES, **(EXT_PROTOTYPES if ext else {})}.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class HconvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hconv status {status}: {msg}")
        self.status = status


def check(lib: C.CDLL, status: int) -> None:
    """Map a status to the reference's exception types (std::invalid_argument -> ValueError)."""
    if status == OK:
        return
    msg = (lib.hconv_last_error() or b"").decode()
    if status == INVALID_ARG:
        raise ValueError(msg)
    if status == UNSUPPORTED:
        raise NotImplementedError(msg)
    raise HconvError(status, msg)
