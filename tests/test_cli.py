"""The verify / tune / bench command line.  CPU: usage errors and the numpy
direct sums that `verify` and the bench spot checks use, pinned to the oracle's
direct_convolution.  GPU: the three subcommands end to end."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import rel_l2

REPO = Path(__file__).resolve().parents[1]


def _cli(*args, env=None):
    return subprocess.run([sys.executable, "-m", "paper_2303_17510_b200", *args], cwd=REPO, capture_output=True,
                          text=True, env={**os.environ, **(env or {})}, timeout=900)


@pytest.mark.parametrize("args", [["verify", "--max-L", "0"], ["bench", "--L", "0"], ["tune", "--L", "x..y"],
                                  ["bench", "--L", "8", "--threads", "2"]])
def test_usage_errors(args):
    r = _cli(*args)
    assert r.returncode == 2, (r.returncode, r.stderr)


def test_direct_sums_match_oracle(oracle):
    from paper_2303_17510_b200.cli import direct

    rng = np.random.default_rng(0)
    for kinds, Ls in [([0], [7]), ([1], [8]), ([2], [9]), ([0, 0], [5, 6]), ([1, 2], [5, 7]), ([1, 1, 2], [4, 6, 9])]:
        shape = [(L + 1) // 2 if k == 2 else L for k, L in zip(kinds, Ls)]
        f = rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)
        g = rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)
        if kinds[-1] == 2:
            if len(Ls) > 1:
                f, g = oracle.symmetrize(Ls, f), oracle.symmetrize(Ls, g)
            else:
                f[0], g[0] = f[0].real, g[0].real
        assert rel_l2(direct(f, g, kinds, Ls), oracle.direct(kinds, Ls, f, g)) < 1e-14


@pytest.mark.gpu
def test_cli_verify_tune_bench(cuda, tmp_path):
    env = {"HCONV_PLAN_CACHE": str(tmp_path / "plans.csv")}
    for kind, dims, maxl in [("complex", 1, 16), ("hermitian", 1, 15), ("centered", 1, 12), ("complex", 2, 6),
                             ("hermitian", 3, 5)]:
        r = _cli("verify", "--kind", kind, "--dims", str(dims), "--max-L", str(maxl), env=env)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "worst relative error" in r.stdout
    r1 = _cli("tune", "--L", "6", "--M", "11", "--copies", "64", "--show-space", env=env)
    assert r1.returncode == 0 and "cached=false" in r1.stdout and "median_ms" in r1.stdout, r1.stdout + r1.stderr
    r2 = _cli("tune", "--L", "6", "--M", "11", "--copies", "64", env=env)
    assert "cached=true" in r2.stdout, r2.stdout
    r = _cli("bench", "--L", "1024", "--M", "2047", "--copies", "64", env=env)
    rows = [l for l in r.stdout.splitlines() if l and not l.startswith("mode")]
    assert r.returncode == 0 and len(rows) >= 3, r.stdout + r.stderr
    strategies = {l.split(",")[4] for l in rows}
    assert {"hybrid", "explicit-pow2"} <= strategies
    for l in rows:
        assert len(l.split(",")) == 7 and float(l.split(",")[5]) > 0
