"""Pin the C restatement of the structure builders (oracle/dpmrf_oracle.c:
orc_region_graph, orc_maximal_cliques) before trusting it.

(1) Known answers of the reference's own tests: proj/tests/graph_test.cpp
    (region graph of a 2x2 block grid, uniform means, single region,
    invariants) and proj/tests/cliques_test.cpp (4-cycle, triangle with a
    tail, isolated vertices, K4, empty graph, lexicographic order).
(2) Bit-for-bit agreement with the reference library (oracle/_ref) on grid,
    brick, random and blob label maps.
"""
import numpy as np
import pytest

from oracle import OracleError, graph_from_edges
from structure_cases import blob_labelmap, grid_labelmap, random_graph_edges, random_labelmap


def _cl(cliques):
    off = [0]
    mem = []
    for c in cliques:
        mem += c
        off.append(len(mem))
    return off, mem


# ---- (1) graph_test.cpp ---------------------------------------------------------
def test_two_by_two_block_grid(orc):  # graph_test.cpp:215-223
    w, h, px, reg, R = grid_labelmap(np.random.default_rng(32), 4, 4, 2)
    g, size = orc.region_graph(w, h, px, reg, R)
    assert g.offsets.tolist() == [0, 2, 4, 6, 8]
    assert g.neighbors.tolist() == [1, 2, 0, 3, 0, 3, 1, 2]
    assert size.tolist() == [4, 4, 4, 4]


def test_uniform_means_exact(orc):  # graph_test.cpp:225-233
    _, _, _, reg, R = grid_labelmap(np.random.default_rng(0), 6, 6, 2)
    g, _ = orc.region_graph(6, 6, np.full(36, 77, np.uint8), reg, R)
    assert (g.region_mean == 77.0).all()


def test_single_region(orc):  # graph_test.cpp:235-244
    w, h, px, reg, R = grid_labelmap(np.random.default_rng(33), 5, 3, 8)
    g, size = orc.region_graph(w, h, px, reg, R)
    assert R == 1 and g.offsets.tolist() == [0, 0] and len(g.neighbors) == 0
    assert size.tolist() == [15]


def test_region_graph_errors(orc):
    with pytest.raises(OracleError):  # num_regions == 0: map not validated (region_graph.cpp:14)
        orc.region_graph(2, 2, np.zeros(4, np.uint8), np.zeros(4, np.uint32), 0)
    with pytest.raises(OracleError):  # id out of range
        orc.region_graph(2, 2, np.zeros(4, np.uint8), np.array([0, 1, 2, 5], np.uint32), 3)
    with pytest.raises(OracleError):  # unused id
        orc.region_graph(2, 2, np.zeros(4, np.uint8), np.array([0, 0, 2, 2], np.uint32), 3)


@pytest.mark.parametrize("seed", range(6))
def test_region_graph_invariants(orc, seed):  # graph_test.cpp:268-298
    rng = np.random.default_rng(36 + seed)
    w, h = int(rng.integers(2, 49)), int(rng.integers(2, 49))
    w, h, px, reg, R = grid_labelmap(rng, w, h, int(rng.integers(1, 8)))
    g, size = orc.region_graph(w, h, px, reg, R)
    assert g.offsets[-1] == len(g.neighbors) and int(size.sum()) == w * h
    for v in range(R):
        nb = g.neighbors[g.offsets[v]:g.offsets[v + 1]]
        assert (np.diff(nb.astype(np.int64)) > 0).all() and v not in nb
        for u in nb:
            assert v in g.neighbors[g.offsets[u]:g.offsets[u + 1]]
    assert float((g.region_mean * size).sum()) == pytest.approx(float(px.astype(np.int64).sum()),
                                                               rel=1e-12)


# ---- (1) cliques_test.cpp --------------------------------------------------------
@pytest.mark.parametrize("n,edges,want", [
    (4, [(0, 1), (0, 2), (1, 3), (2, 3)], [[0, 1], [0, 2], [1, 3], [2, 3]]),  # :94-98
    (4, [(0, 1), (0, 2), (1, 2), (2, 3)], [[0, 1, 2], [2, 3]]),              # :100-104
    (3, [], [[0], [1], [2]]),                                                # :106-110
    (4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)], [[0, 1, 2, 3]]),   # :112-117
    (0, [], []),                                                             # :119-123
])
def test_cliques_known_answers(orc, n, edges, want):
    off, mem = orc.maximal_cliques(graph_from_edges(n, edges))
    assert (off.tolist(), mem.tolist()) == _cl(want)


def test_cliques_lexicographic(orc):  # cliques_test.cpp:130-145
    rng = np.random.default_rng(41)
    g = graph_from_edges(12, random_graph_edges(rng, 12, 0.4))
    off, mem = orc.maximal_cliques(g)
    cl = [mem[off[c]:off[c + 1]].tolist() for c in range(len(off) - 1)]
    assert all(c == sorted(c) for c in cl) and cl == sorted(cl)


# ---- (2) against the reference itself ---------------------------------------------
def _cases():
    rng = np.random.default_rng(7)
    return [("grid", grid_labelmap(rng, 96, 80, 8)), ("grid_ragged", grid_labelmap(rng, 61, 47, 5)),
            ("brick", grid_labelmap(rng, 96, 80, 8, brick=True)),
            ("random", random_labelmap(rng, 50, 40, 600)), ("random_dense", random_labelmap(rng, 30, 30, 12)),
            ("blob", blob_labelmap(rng, 120, 90))]


@pytest.mark.parametrize("name,case", _cases(), ids=[c[0] for c in _cases()])
def test_structure_vs_ref(orc, ref, name, case):
    w, h, px, reg, R = case
    g, size = orc.region_graph(w, h, px, reg, R)
    p = ref.labelmap(w, h, px, reg, R)
    gr = p.graph()
    assert np.array_equal(g.offsets, gr.offsets) and np.array_equal(g.neighbors, gr.neighbors)
    assert np.array_equal(g.region_mean, gr.region_mean)
    off, mem = orc.maximal_cliques(g)
    ro, rm = p.cliques()
    assert np.array_equal(off, ro) and np.array_equal(mem, rm)


@pytest.mark.parametrize("n,p", [(12, 0.4), (20, 0.5), (40, 0.2), (60, 0.1)])
def test_cliques_random_graphs_vs_ref(orc, ref, n, p):
    rng = np.random.default_rng(n)
    g = graph_from_edges(n, random_graph_edges(rng, n, p))
    off, mem = orc.maximal_cliques(g)
    ro, rm = ref.arrays(g).cliques()
    assert np.array_equal(off, ro) and np.array_equal(mem, rm)
