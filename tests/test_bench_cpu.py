"""bench.py launch logic and the per-rank HBM budget, on CPU.

`bench.py --gpus N` must run N ranks (one per GPU) even without a launcher:
it spawns them through torch.distributed.run.  The dry mode runs the same
launch, rendezvous and max-over-ranks timing on gloo without kernels.
"""

import json
import os
import subprocess
import sys

import pytest

from paper_1904_03057_b200.device import heat_memory_plan
from paper_1904_03057_b200.errors import ConfigurationError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          capture_output=True, text=True, timeout=300, env=e, cwd=ROOT)


@pytest.mark.parametrize("n", [2, 3])
def test_bench_gpus_flag_spawns_ranks(n):
    res = _bench("--gpus", str(n), "--dry", "--steps", "2", "--warmup", "0")
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == n and line["dry"] is True
    assert line["planes_covered"] == 930  # the slabs tile the global z axis
    assert line["config"]["parallelism"] == f"zslab{n}"


def test_bench_rejects_gpus_world_mismatch():
    res = _bench("--gpus", "1", "--dry", env={"WORLD_SIZE": "2", "RANK": "0"})
    assert res.returncode != 0
    assert "WORLD_SIZE" in res.stderr


def test_memory_plan_fits_c5():
    """C5's strong-scaling anchor 1536^3 (p = 3) fits one B200: u, F, r, Ap
    (b shares Ap) and the two-field search-direction ring = 6 fields."""
    plan = heat_memory_plan((1536,) * 3, 3, world=1)
    assert plan["ring"] == 2 and plan["fields"] == 6
    assert plan["bytes"] <= 175e9
    # the 1024^3-per-GPU weak-scaling size and C3 (930^3): 6 fields as well
    assert heat_memory_plan((1024,) * 3, 3, 1)["bytes"] < 55e9
    assert heat_memory_plan((8 * 1024, 1024, 1024), 3, 8)["bytes"] < 55e9
    c3 = heat_memory_plan((930,) * 3, 3, 1)
    assert c3["fields"] == 6 and c3["bytes"] < 40e9
    with pytest.raises(ConfigurationError):
        heat_memory_plan((2048,) * 3, 3, 1)
