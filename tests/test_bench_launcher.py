"""CPU: `python bench.py --gpus N` launches its own ranks when no launcher set WORLD_SIZE (one
process per GPU through torch.distributed.run on 127.0.0.1), the ranks rendezvous and agree on
the workload, and rank 0 alone prints the line.  --dry-run stops before the GPU work (gloo)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", *args],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 only
    return json.loads(lines[0])


@pytest.mark.parametrize("n,grid", [(1, [256, 256, 256]), (2, [512, 256, 256]),
                                    (4, [512, 512, 256])])
def test_weak_scaling_launcher(n, grid):
    line = _run("--gpus", str(n))
    assert line["n_gpus"] == n
    assert line["config"]["grid"] == grid  # SURVEY §8(d) weak-scaling grids
    assert line["rows_covered"] == grid[0] * grid[1] * grid[2] == line["config"]["n"]


def test_strong_scaling_launcher():
    line = _run("--gpus", "2", "--config", "c5", "--scaling", "strong")
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["grid"] == [512, 512, 512]
    assert line["config"]["nnz"] == 937951232
