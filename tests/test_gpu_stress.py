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
