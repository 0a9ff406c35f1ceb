"""bench.py's N>1 launch as the driver may invoke it (no torchrun in front):
it re-launches itself one process per GPU under torch.distributed.run, and
`--dry-run` stops after the gloo rendezvous with every rank's placement.
Checked against the reference geometry (grid.cpp:43-61: rank = k q^2 + i q
+ j) and the synthetic-weight seeding (depth replicas of a TesseractB
block share a seed)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dry_run(gpus):
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(gpus), "--dry-run"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus,grid,q", [(2, "[1,1,2]", 1), (8, "[2,2,2]", 2)])
def test_bench_spawns_one_rank_per_gpu(gpus, grid, q):
    out = _dry_run(gpus)
    assert out["world"] == gpus
    ranks = sorted(out["ranks"], key=lambda r: r["rank"])
    assert [r["rank"] for r in ranks] == list(range(gpus))
    for r in ranks:
        i, j, k = r["coord"]
        assert r["grid"] == grid
        assert r["device"] == r["local_rank"] == r["rank"] == k * q * q + i * q + j
    # weights: one seed per (i, j), shared by the depth replicas; activations per rank
    by_ij = {}
    for r in ranks:
        i, j, _ = r["coord"]
        by_ij.setdefault((i, j), set()).add(r["seeds"]["weight"])
    assert all(len(v) == 1 for v in by_ij.values())
    assert len({r["seeds"]["activation"] for r in ranks}) == gpus
    assert len({next(iter(v)) for v in by_ij.values()}) == q * q
