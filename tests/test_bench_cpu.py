"""bench.py host logic on CPU: the self-launch under torch.distributed.run for --gpus N, the
workload identity both arms print, the L2 rotation and the algorithmic figures of SURVEY §8(d)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import bench  # noqa: E402


def test_self_launch_spawns_one_rank_per_gpu():
    out = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--launch-check"],
                         capture_output=True, text=True, timeout=300, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = []
    for l in out.stdout.splitlines():  # the launcher may add lines of its own
        if l.startswith("{"):
            try:
                d = json.loads(l)
            except ValueError:
                continue
            if isinstance(d, dict) and "rank" in d:
                lines.append(d)
    assert sorted(l["rank"] for l in lines) == [0, 1]
    assert all(l["world"] == 2 for l in lines)
    assert sorted(l["local"] for l in lines) == [0, 1]
    assert all(l["config"] == "c5" for l in lines)  # the partitioned 3D config above one GPU


def test_single_gpu_defaults_to_config2():
    out = subprocess.run([sys.executable, str(REPO / "bench.py"), "--launch-check"], capture_output=True, text=True,
                         timeout=120, cwd=REPO)
    assert json.loads(out.stdout.strip().splitlines()[-1]) == {"rank": 0, "world": 1, "local": 0, "config": "c2"}


@pytest.mark.parametrize("name", sorted(bench.CONFIGS))
def test_config_dict_is_implementation_free(name):
    d = bench.config_dict(name)
    assert set(d) == {"workload", "config", "global_batch", "l2"}
    assert d == bench.config_dict(name)  # both arms call the same function


def test_l2_rotation():
    for name in bench.CONFIGS:
        sets = bench.input_sets(name)
        assert sets * bench.working_set(name) >= 2 * bench.L2_BYTES
    assert bench.input_sets("c1") > 1 and bench.input_sets("c2") == 1


def test_algorithmic_figures_match_survey():
    # bytes_alg and flops_alg per configuration
    want = {"c1": (50331648, 3.584e8), "c2": (1179648000, 1.0285e10), "c3": (805306368, 5.556e9),
            "c4": (201326592, 4.629e9), "c5": (3208654848, 6.874e10)}
    for name, (b, f) in want.items():
        nb, nf = bench.algorithmic(name)
        assert nb == b
        assert abs(nf - f) / f < 2e-3, (name, nf, f)
