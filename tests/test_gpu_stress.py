"""Synchronisation stress of every kernel family (tools/stress_cases.py): NaN-poisoned scratch,
persistent loops with several lines per CTA, bit-identical repeated runs, oracle parity.  Each
case runs in its own process (the library reads HCONV_* once per process)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO / "tools"))


def _cases():
    import stress_cases

    return sorted(stress_cases.CASES)


@pytest.mark.parametrize("case", _cases())
def test_stress_case(cuda, case):
    env = dict(os.environ, HCONV_POISON="1")
    r = subprocess.run([sys.executable, str(REPO / "tools" / "stress_cases.py"), case], capture_output=True,
                       text=True, timeout=600, env=env, cwd=REPO)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "bit-identical" in r.stdout


@pytest.mark.parametrize("case", ["cols_2d", "cols_3d_herm", "cols_3d_c5_like", "cols_2d_4096", "cols_2d_2048"])
def test_tma_column_tiles_bit_identical(cuda, case, tmp_path):
    """The tensor-map TMA column kernels (two tile buffers, or one buffer plus staged rows for the
    long blocks) move the same tiles as the cp.async / plain-load kernels: identical arithmetic, so
    identical bits (HCONV_NO_COLS_TMA=1 selects the non-TMA path)."""
    outs = []
    for flag in ("0", "1"):
        env = dict(os.environ, HCONV_NO_COLS_TMA=flag)
        pre = str(tmp_path / f"o{flag}")
        r = subprocess.run([sys.executable, str(REPO / "tools" / "stress_cases.py"), "--dump", pre, case],
                           capture_output=True, text=True, timeout=600, env=env, cwd=REPO)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
        import numpy as np

        outs.append(np.load(f"{pre}_{case}.npy"))
    assert (outs[0] == outs[1]).all()
