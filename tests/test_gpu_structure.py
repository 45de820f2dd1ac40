"""Device structure builders (csrc/structure.cu) vs the oracle, bit for bit.

build_region_graph (region_graph.cpp:10-73) and enumerate_maximal_cliques
(cliques.cpp:53-106) on the device must equal orc_region_graph /
orc_maximal_cliques (pinned to the reference in test_oracle_structure.py):
same CSR, same means (integer sums / sizes, one division), same cliques in
the same canonical order.  The device-resident pipeline (graph -> cliques ->
neighborhoods -> optimize) must equal the host-input pipeline.
"""
import numpy as np
import pytest

from oracle import graph_from_edges
from structure_cases import blob_labelmap, grid_labelmap, random_graph_edges, random_labelmap

pytestmark = pytest.mark.gpu
E = pytest.importorskip("paper_1809_05018_b200.engine")
from paper_1809_05018_b200 import inputs  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = E.Context(0)
    yield c
    c.close()


def _graph_equal(ctx, orc, case):
    w, h, px, reg, R = case
    A = ctx.build_region_graph(w, h, px, reg, R)
    got = ctx.get_graph()
    want, size = orc.region_graph(w, h, px, reg, R)
    assert A == len(want.neighbors)
    assert np.array_equal(got.offsets, want.offsets)
    assert np.array_equal(got.neighbors, want.neighbors)
    assert np.array_equal(got.region_mean.view(np.uint64), want.region_mean.view(np.uint64))
    assert np.array_equal(got.region_size, size)
    return want


def _cliques_equal(ctx, orc, g):
    C, CS = ctx.enumerate_maximal_cliques()
    got = ctx.get_cliques()
    off, mem = orc.maximal_cliques(g)
    assert (C, CS) == (len(off) - 1, len(mem))
    assert np.array_equal(got.offsets, off) and np.array_equal(got.members, mem)
    return off, mem


def _cases():
    rng = np.random.default_rng(11)
    return [
        ("2x2_blocks", grid_labelmap(rng, 4, 4, 2)),
        ("single_region", grid_labelmap(rng, 5, 3, 8)),
        ("one_pixel_regions", grid_labelmap(rng, 3, 2, 1)),
        ("one_row", grid_labelmap(rng, 77, 1, 3)),
        ("one_column", grid_labelmap(rng, 1, 45, 4)),
        ("grid_ragged", grid_labelmap(rng, 61, 47, 5)),
        ("grid_multi_tile", grid_labelmap(rng, 300, 170, 7)),
        ("brick", grid_labelmap(rng, 200, 136, 8, brick=True)),
        ("random", random_labelmap(rng, 50, 40, 600)),
        ("random_dense", random_labelmap(rng, 30, 30, 12)),
        ("random_tiles", random_labelmap(rng, 130, 70, 3000)),
        ("blob_long_lists", blob_labelmap(rng, 260, 200)),  # background degree > 1024
    ]


@pytest.mark.parametrize("name,case", _cases(), ids=[c[0] for c in _cases()])
def test_region_graph_and_cliques(ctx, orc, name, case):
    g = _graph_equal(ctx, orc, case)
    _cliques_equal(ctx, orc, g)


def test_blob_case_exercises_long_segments(orc):
    w, h, px, reg, R = blob_labelmap(np.random.default_rng(11), 260, 200)
    g, _ = orc.region_graph(w, h, px, reg, R)
    assert g.offsets[1] - g.offsets[0] > 1024  # background region's list


@pytest.mark.parametrize("brick", [False, True])
def test_phantom_slices(ctx, orc, brick):
    sl = inputs.synthetic_slice(512, 8, brick=brick, seed=5)
    g = _graph_equal(ctx, orc, (512, 512, sl.image, sl.region, sl.graph.num_vertices))
    off, mem = _cliques_equal(ctx, orc, g)
    # and the host input builder (what bench/tests feed the optimizer) agrees
    assert np.array_equal(sl.cliques.offsets, off) and np.array_equal(sl.cliques.members, mem)


def test_config_b_slice(ctx):
    """Full 2560^2 slice: device graph + cliques == the host builder's (itself
    bit-identical to the reference, test_oracle.py)."""
    sl = inputs.synthetic_slice(2560, 8, seed=42)
    ctx.build_region_graph(2560, 2560, sl.image, sl.region, sl.graph.num_vertices)
    got = ctx.get_graph()
    assert np.array_equal(got.offsets, sl.graph.offsets)
    assert np.array_equal(got.neighbors, sl.graph.neighbors)
    assert np.array_equal(got.region_mean, sl.graph.region_mean)
    ctx.enumerate_maximal_cliques()
    cl = ctx.get_cliques()
    assert np.array_equal(cl.offsets, sl.cliques.offsets)
    assert np.array_equal(cl.members, sl.cliques.members)


@pytest.mark.parametrize("n,edges", [
    (4, [(0, 1), (0, 2), (1, 3), (2, 3)]),               # cliques_test.cpp:94-98
    (4, [(0, 1), (0, 2), (1, 2), (2, 3)]),               # :100-104
    (3, []),                                             # :106-110
    (4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]),  # :112-117
    (0, []),                                             # :119-123
])
def test_cliques_known_answers(ctx, orc, n, edges):
    g = graph_from_edges(n, edges)
    ctx.set_graph(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
    _cliques_equal(ctx, orc, g)


@pytest.mark.parametrize("n,p", [(12, 0.4), (20, 0.5), (40, 0.2), (60, 0.1), (300, 0.02)])
def test_cliques_random_graphs(ctx, orc, n, p):
    rng = np.random.default_rng(n)
    g = graph_from_edges(n, random_graph_edges(rng, n, p))
    ctx.set_graph(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
    _cliques_equal(ctx, orc, g)


def test_errors(ctx):
    z8, z32 = np.zeros(4, np.uint8), np.zeros(4, np.uint32)
    with pytest.raises(E.InputError):       # num_regions == 0 (region_graph.cpp:14)
        ctx.build_region_graph(2, 2, z8, z32, 0)
    with pytest.raises(IndexError):         # id >= num_regions
        ctx.build_region_graph(2, 2, z8, np.array([0, 1, 2, 5], np.uint32), 3)
    with pytest.raises(E.InputError):       # unused id: the map was not validated
        ctx.build_region_graph(2, 2, z8, np.array([0, 0, 2, 2], np.uint32), 3)
    with pytest.raises(E.InputError):       # image / map dimensions differ
        ctx.build_region_graph(3, 2, z8, z32, 1)
    # the context stays usable
    ctx.build_region_graph(2, 2, z8, z32, 1)
    assert ctx.get_graph().offsets.tolist() == [0, 0]


def test_device_pipeline_optimize(ctx, orc):
    """image + label map -> graph -> cliques -> hoods -> optimize, all resident,
    equals optimize over the host-built inputs."""
    sl = inputs.synthetic_slice(384, 8, seed=9)
    ctx.build_region_graph(384, 384, sl.image, sl.region, sl.graph.num_vertices)
    ctx.enumerate_maximal_cliques()
    ctx.build_neighborhoods_resident()
    cfg = E.OptimizerConfig(rng_seed=9, em_max_iters=6)
    got = ctx.optimize(cfg, trace_level=E.TRACE_EM)
    ref = E.Context(0)
    try:
        ref.set_graph(sl.graph)
        ref.build_neighborhoods(sl.cliques)
        want = ref.optimize(cfg, trace_level=E.TRACE_EM)
    finally:
        ref.close()
    assert np.array_equal(got.labels, want.labels)
    assert np.array_equal(got.mu, want.mu) and np.array_equal(got.sigma, want.sigma)
    assert [e.total_energy for e in got.trace] == [e.total_energy for e in want.trace]
