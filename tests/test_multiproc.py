"""N>1 host path on CPU with world_size-2 and -8 gloo process groups: the
launcher-side plumbing bench.py uses (rank -> grid coordinate, the 128-byte
NCCL unique-id exchange, max-over-ranks timing) and the communicator split
plan libtess hands to ncclCommSplit (color = group_index, key = slot; ref
grid.cpp:79-95), checked against the reference geometry."""
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_14500_b200.launch import GRIDS, free_port as _free_port


def _worker(rank, world, port, q, d, allow, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import paper_2105_14500_b200 as tess
    grid = tess.GridSpec(q, d, allow)
    c = grid.coord_of(rank)
    # split plan per family: (color, key)
    plan = [(grid.group_index(c, f), grid.slot_in_group(c, f)) for f in (0, 1, 2)]
    gathered = [None] * world
    dist.all_gather_object(gathered, plan)
    # unique-id exchange exactly as bench.py does it
    blob = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(blob, src=0)
    # max over ranks
    t = torch.tensor([float(rank)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ok = blob[0] == bytes(range(128)) and t.item() == world - 1
        for f in (0, 1, 2):
            colors = {}
            for r in range(world):
                colors.setdefault(gathered[r][f][0], []).append((gathered[r][f][1], r))
            for members in colors.values():
                members.sort()
                ranks = [r for _, r in members]
                keys = [k for k, _ in members]
                ok &= keys == list(range(len(members)))
                want = [grid.rank_of(m) for m in grid.group_of(grid.coord_of(ranks[0]), f)]
                ok &= ranks == want
                ok &= len(members) == grid.group_size(f)
        out.put(ok)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_split_plan_and_launcher_plumbing(world):
    q, d, allow = GRIDS[world]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), q, d, allow, out), nprocs=world,
                       join=True, start_method="spawn")
    assert out.get(timeout=30) is True


def test_row_pairs_match_survey_8e():
    import paper_2105_14500_b200 as tess
    g = tess.GridSpec(2, 2)
    pairs = {f: sorted({tuple(sorted(g.rank_of(m) for m in g.group_of(g.coord_of(r), f)))
                        for r in range(8)}) for f in (0, 1, 2)}
    assert pairs[0] == [(0, 1), (2, 3), (4, 5), (6, 7)]
    assert pairs[1] == [(0, 2), (1, 3), (4, 6), (5, 7)]
    assert pairs[2] == [(0, 4), (1, 5), (2, 6), (3, 7)]
