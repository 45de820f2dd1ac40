"""Multi-GPU placement for the optimization phase (host logic).

Two ways the path shards:

* **slice stacks** (config E): independent slices, each with its own
  parameters and convergence state (the reference processes a volume as
  independent 2-D slices).  Slices are dealt to ranks
  round-robin; no collective touches the data path -- ranks only agree on
  timing (max) and totals (sum).
* **one giant slice** (config D): contiguous vertex ranges (multiples of the
  256-vertex tile) and contiguous series ranges (multiples of the 1024-element
  fold leaf), equal-sized so the per-EM allgathers are plain in-place
  allgathers.  ``partition_bounds`` / ``halo_windows`` restate the plan of
  csrc/partition.cu (plan(), k_halo_plan): per (source, destination) pair the
  [lo, hi] window of source-owned vertices whose labels the destination's
  vertex pass reads and whose minima its hood pass folds.
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


@dataclass
class PartitionPlan:
    world: int
    chunk_v: int            # vertices per partition (multiple of 256)
    chunk_h: int            # series per partition (multiple of 1024)
    vb: np.ndarray          # world+1 vertex boundaries
    hb: np.ndarray          # world+1 series boundaries
    lab_win: np.ndarray     # [world, world, 2] (lo, hi) source -> destination; lo > hi = none
    min_win: np.ndarray     # [world, world, 2]

    def halo_bytes(self, rank: int = -1) -> int:
        """Bytes of labels + minima sent per MAP iteration by ``rank`` (-1: all)."""
        n = 0
        for s in range(self.world):
            if rank >= 0 and s != rank:
                continue
            for d in range(self.world):
                for win, size in ((self.lab_win, 1), (self.min_win, 8)):
                    lo, hi = int(win[s, d, 0]), int(win[s, d, 1])
                    if lo <= hi:
                        n += size * (hi - lo + 1)
        return n


def partition_bounds(num_vertices: int, num_series: int, world: int, tile: int = 256,
                     leaf: int = 1024):
    """Equal-chunk vertex and series ranges of partition.cu plan()."""
    if world < 1:
        raise ValueError("world must be >= 1")
    cv = -(-num_vertices // world)
    chunk_v = max(tile, -(-cv // tile) * tile)
    ch = -(-num_series // world)
    chunk_h = max(leaf, -(-ch // leaf) * leaf)
    vb = np.minimum(np.arange(world + 1, dtype=np.int64) * chunk_v, num_vertices)
    hb = np.minimum(np.arange(world + 1, dtype=np.int64) * chunk_h, num_series)
    return chunk_v, chunk_h, vb, hb


def _owner(bounds, x):
    # largest r with bounds[r] <= x (the device's binary search)
    return np.searchsorted(bounds[:-1], x, side="right") - 1


def halo_windows(offsets, neighbors, series_offsets, members, world: int) -> PartitionPlan:
    """Plan of a vertex-range partition over the nonempty-hood series."""
    offsets = np.asarray(offsets, np.int64)
    neighbors = np.asarray(neighbors, np.int64)
    series_offsets = np.asarray(series_offsets, np.int64)
    members = np.asarray(members, np.int64)
    R = len(offsets) - 1
    Hs = len(series_offsets) - 1
    chunk_v, chunk_h, vb, hb = partition_bounds(R, Hs, world)
    lab = np.empty((world, world, 2), np.int64)
    mn = np.empty((world, world, 2), np.int64)
    lab[..., 0] = mn[..., 0] = 0xFFFFFFFF
    lab[..., 1] = mn[..., 1] = 0
    deg = np.diff(offsets)
    dst = _owner(vb, np.repeat(np.arange(R), deg))
    src = _owner(vb, neighbors)
    _windows(lab, src, dst, neighbors, world)
    sz = np.diff(series_offsets)
    dst = _owner(hb, np.repeat(np.arange(Hs), sz))
    src = _owner(vb, members[series_offsets[0]:series_offsets[-1]] if Hs else members[:0])
    _windows(mn, src, dst, members[series_offsets[0]:series_offsets[-1]] if Hs else members[:0],
             world)
    return PartitionPlan(world, chunk_v, chunk_h, vb, hb, lab, mn)


def _windows(win, src, dst, ids, world):
    cross = src != dst
    key = src[cross] * world + dst[cross]
    val = ids[cross]
    if not len(val):
        return
    flat = win.reshape(world * world, 2)
    np.minimum.at(flat[:, 0], key, val)
    np.maximum.at(flat[:, 1], key, val)
