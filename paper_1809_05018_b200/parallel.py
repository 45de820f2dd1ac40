"""Multi-GPU placement for the optimization phase (host logic).

Two ways the path shards:

* **slice stacks** (config E): independent slices, each with its own
  parameters and convergence state (the reference processes a volume as
  independent 2-D slices).  Slices are dealt to ranks
  round-robin; no collective touches the data path -- ranks only agree on
  timing (max) and totals (sum).
* **one giant slice** (config D): contiguous vertex ranges per rank; each rank
  owns the hoods whose smallest member it owns (cliques are lexicographically
  sorted, so owned hoods are contiguous).  ``halo_plan`` computes, per rank,
  the foreign vertices whose labels / minima it must receive each MAP
  iteration.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np


def shard_slices(num_slices: int, world: int, rank: int) -> List[int]:
    """Round-robin deal of slice indices (slice z -> rank z % world)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return list(range(rank, num_slices, world))


def vertex_ranges(num_vertices: int, world: int) -> np.ndarray:
    """world+1 boundaries of contiguous, balanced vertex ranges."""
    return np.array([(num_vertices * r) // world for r in range(world + 1)], dtype=np.int64)


@dataclass
class HaloPlan:
    lo: int                 # owned vertex range [lo, hi)
    hi: int
    hood_lo: int            # owned hood range [hood_lo, hood_hi)
    hood_hi: int
    label_halo: np.ndarray  # foreign vertices whose labels the owned vertices read (discord)
    minE_halo: np.ndarray   # foreign vertices whose minima the owned hoods fold


def halo_plan(offsets, neighbors, hood_offsets, hood_members, world: int, rank: int) -> HaloPlan:
    """Ownership and halo sets of ``rank`` for a vertex-range partition."""
    offsets = np.asarray(offsets, np.int64)
    neighbors = np.asarray(neighbors, np.int64)
    hood_offsets = np.asarray(hood_offsets, np.int64)
    hood_members = np.asarray(hood_members, np.int64)
    R = len(offsets) - 1
    b = vertex_ranges(R, world)
    lo, hi = int(b[rank]), int(b[rank + 1])
    H = len(hood_offsets) - 1
    first = np.full(H, -1, np.int64)
    nonempty = hood_offsets[1:] > hood_offsets[:-1]
    first[nonempty] = hood_members[hood_offsets[:-1][nonempty]]
    owner = np.searchsorted(b, first, side="right") - 1
    owner[~nonempty] = -1
    mine = np.nonzero(owner == rank)[0]
    hood_lo = int(mine[0]) if len(mine) else 0
    hood_hi = int(mine[-1]) + 1 if len(mine) else 0
    if len(mine) and not np.all(np.diff(mine) == 1):
        raise ValueError("owned hoods are not contiguous (cliques not lexicographic?)")
    nb = neighbors[offsets[lo]:offsets[hi]]
    label_halo = np.unique(nb[(nb < lo) | (nb >= hi)])
    hm = hood_members[hood_offsets[hood_lo]:hood_offsets[hood_hi]] if len(mine) else hood_members[:0]
    minE_halo = np.unique(hm[(hm < lo) | (hm >= hi)])
    return HaloPlan(lo, hi, hood_lo, hood_hi, label_halo, minE_halo)
