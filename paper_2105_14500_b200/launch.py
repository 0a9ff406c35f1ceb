"""One-process-per-GPU launch plumbing shared by bench.py and the tests.

The reference runs every rank of a [q,q,d] grid as a std::thread of one
process (runtime.cpp:534-554); on B200 each rank is a process bound to one
GPU (device = local rank = k*q^2 + i*q + j on one node). This module holds
the host-side pieces of that launch:

* `spawn(script, argv, nproc)`: re-launch `script` under
  torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1) when
  the caller was started without it, forwarding the exit status;
* `rank_env()`: (rank, local_rank, world) from the torchrun environment;
* `grid_for(world)`: the [q,q,d] grid bench.py maps N GPUs to;
* `seeds(grid, rank)`: per-tensor seeds for synthetic data that respect the
  Tesseract layouts -- activations differ per rank (TesseractA blocks),
  weight blocks depend on (i, j) only (TesseractB blocks are replicated over
  depth, shard.cpp:80-98), LayerNorm vectors on j only (the j-slice
  replicated over (i, k), layers.cpp:140-166).
"""
import os
import socket
import subprocess
import sys

# N GPUs -> (q, d, allow_d_gt_q): [1,1,1], [1,1,2], [2,2,1], [2,2,2]
GRIDS = {1: (1, 1, True), 2: (1, 2, True), 4: (2, 1, False), 8: (2, 2, False)}


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def rank_env():
    """(rank, local_rank, world) of this process (1-process default)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def spawn(script: str, argv, nproc: int) -> int:
    """Run `script argv` as `nproc` ranks under torch.distributed.run on this
    node; returns the launcher's exit status (rank 0's stdout passes through)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", script, *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def grid_for(world: int):
    if world not in GRIDS:
        raise SystemExit(f"--gpus must be one of {sorted(GRIDS)}")
    return GRIDS[world]


def seeds(grid, rank: int, base: int = 1234) -> dict:
    """Seeds per synthetic tensor family for `rank` of `grid` (a GridSpec)."""
    c = grid.coord_of(rank)
    q = grid.q()
    return {"activation": base + 1000 + rank,        # x, dy: this rank's TesseractA block
            "weight": base + 2000 + c.i * q + c.j,   # TesseractB block (i, j), all k
            "ln": base + 3000 + c.j}                 # LayerNorm j-slice, all (i, k)
