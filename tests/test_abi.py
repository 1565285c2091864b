"""The C-ABI libraries load and export every symbol the headers declare (no compute calls)."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2303_17510_b200 import _abi

REPO = Path(__file__).resolve().parents[1]


def _declared(header):
    txt = (REPO / "include" / header).read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hconv_[a-z_]+)\s*\(", txt)))


def test_prototypes_cover_header():
    assert _declared("hconv.h") == sorted(_abi.PROTOTYPES)
    assert _declared("hconv_ext.h") == sorted(_abi.EXT_PROTOTYPES)


def test_cuda_library_exports_all():
    from paper_2303_17510_b200 import hconv

    if not hconv.LIB_PATH.exists():
        pytest.fail("libhconv_cuda.so not built (run __graft_entry__.build())")
    lib = C.CDLL(str(hconv.LIB_PATH))
    for name in _declared("hconv.h") + _declared("hconv_ext.h"):
        assert hasattr(lib, name), name
    _abi.bind(lib, ext=True)
    assert lib.hconv_backend() == b"cuda-sm_100a"


def test_oracle_library_exports_all(oracle):
    for name in _declared("hconv.h"):
        assert hasattr(oracle.lib, name), name
    assert oracle.lib.hconv_backend() == b"oracle-cpu"


def test_cuda_library_plan_functions_without_gpu():
    """Host-only entry points work on a CPU box (pure C++ behind the ABI)."""
    from paper_2303_17510_b200 import hconv

    pp = hconv.deriveParams(6, 11, 4)
    assert (pp.p, pp.q, pp.n, pp.regime) == (2, 3, 3, hconv.Regime.P2)
    with pytest.raises(ValueError):
        hconv.deriveParams(0, 1, 1)
