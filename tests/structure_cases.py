"""Image + label-map cases for the structure builders (region graph, cliques).

random_labelmap: every pixel draws a region id (every id used) -- fragmented
regions, high degrees, dense clique structure.  blob_labelmap: one background
region around many small square regions -- the background's adjacency list is
long (exercises the >1024-key sort path on the device).
"""
import numpy as np


def random_labelmap(rng, w, h, R):
    reg = rng.integers(0, R, w * h).astype(np.uint32)
    reg[:R] = np.arange(R, dtype=np.uint32)  # every id used
    px = rng.integers(0, 256, w * h).astype(np.uint8)
    return w, h, px, reg, R


def blob_labelmap(rng, w, h, step=4, size=2):
    reg = np.zeros((h, w), np.uint32)
    nxt = 1
    for y in range(1, h - size, step):
        for x in range(1, w - size, step):
            reg[y:y + size, x:x + size] = nxt
            nxt += 1
    px = rng.integers(0, 256, w * h).astype(np.uint8)
    return w, h, px, reg.reshape(-1), nxt


def grid_labelmap(rng, w, h, block, brick=False):
    from paper_1809_05018_b200 import inputs
    reg, R = inputs.oversegment(w, h, block, brick)
    px = rng.integers(0, 256, w * h).astype(np.uint8)
    return w, h, px, reg, R


def edges_graph(n, edges):
    from oracle import graph_from_edges
    return graph_from_edges(n, edges)


def random_graph_edges(rng, n, p):
    """random_graph of proj/tests/cliques_test.cpp:41-50 (edge a<b with probability p)."""
    return [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < p]
