"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic:
slice dealing, max/sum agreement of the bench's timing, and the vertex-range
halo plan of a giant slice."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1809_05018_b200.parallel import shard_slices
    mine = shard_slices(64, world, rank)
    # each rank "times" its shard; the job time is the max, the work the sum
    t = torch.tensor([float(len(mine)) * (1.0 + rank)], dtype=torch.float64)
    n = torch.tensor([float(len(mine))], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    out[rank] = (t.item(), n.item(), gathered)
    dist.destroy_process_group()


def test_slice_sharding_two_ranks():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        t, n, gathered = res[rank]
        assert n == 64.0
        assert t == 32.0 * 2.0
        flat = sorted(z for part in gathered for z in part)
        assert flat == list(range(64))  # every slice exactly once


def test_halo_plan_grid_graph():
    from oracle import C, graph_from_edges
    # 6x6 grid of regions, edge cliques, hoods from the oracle's build
    n = 6
    edges = [(r * n + c, r * n + c + 1) for r in range(n) for c in range(n - 1)]
    edges += [(r * n + c, (r + 1) * n + c) for r in range(n - 1) for c in range(n)]
    g = graph_from_edges(n * n, edges)
    cl = sorted(tuple(sorted(e)) for e in edges)
    c_off = np.arange(0, 2 * len(cl) + 1, 2, dtype=np.uint32)
    hoods, _ = C().build_neighborhoods(g, c_off, np.array(cl, np.uint32).ravel())
    from paper_1809_05018_b200.parallel import halo_plan, vertex_ranges
    world = 3
    b = vertex_ranges(n * n, world)
    owned = []
    for r in range(world):
        p = halo_plan(g.offsets, g.neighbors, hoods.offsets, hoods.members, world, r)
        assert (p.lo, p.hi) == (b[r], b[r + 1])
        owned += list(range(p.hood_lo, p.hood_hi))
        # discord of owned vertices needs exactly the foreign neighbors
        need = set()
        for v in range(p.lo, p.hi):
            need |= {int(u) for u in g.neighbors[g.offsets[v]:g.offsets[v + 1]]
                     if not (p.lo <= u < p.hi)}
        assert set(p.label_halo.tolist()) == need
        # grid: halo is at most one block row on each side
        assert len(p.label_halo) <= 2 * n
        # hoods are owned by their smallest member: their halo lies above the range
        assert all(p.hi <= v < p.hi + 3 * n for v in p.minE_halo)
    assert owned == list(range(hoods.size))  # every hood owned once, in order
