"""Step functions of engine.hpp on the device vs the oracle (and the
reference's own golden vectors, proj/tests/mrf_engine_test.cpp)."""
import numpy as np
import pytest

from oracle import Hoods, graph_from_edges, random_graph

pytestmark = pytest.mark.gpu
E = pytest.importorskip("paper_1809_05018_b200.engine")

WORKED = (np.array([0, 4, 7], np.uint32), np.array([0, 1, 2, 5, 1, 3, 4], np.uint32))


@pytest.fixture(scope="module")
def ctx():
    c = E.Context(0)
    yield c
    c.close()


def test_replication_and_slot_map(ctx):  # mrf_engine_test.cpp:132-184
    ctx.set_hoods(E.NeighborhoodSet(*WORKED))
    rep = ctx.replicate_by_label(2)
    assert rep.test_label.tolist() == [0, 0, 0, 0, 1, 1, 1, 1, 0, 0, 0, 1, 1, 1]
    assert rep.old_index.tolist() == [0, 1, 2, 3, 0, 1, 2, 3, 4, 5, 6, 4, 5, 6]
    assert rep.hood_id.tolist() == [0] * 8 + [1] * 6
    assert ctx.slot_hood_map().tolist() == [0, 0, 0, 0, 1, 1, 1]
    ctx.set_hoods(E.NeighborhoodSet(np.array([0], np.uint32), np.zeros(0, np.uint32)))
    assert len(ctx.replicate_by_label(2).test_label) == 0


def test_discord_energies_mins(ctx, orc):
    g = graph_from_edges(4, [(0, 1), (0, 2), (1, 2), (2, 3)])
    ctx.set_graph(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
    assert ctx.discord_counts([0, 1, 1, 0], 2).tolist() == [2, 1, 1, 1, 0, 1, 2, 0]
    ctx.set_hoods(E.NeighborhoodSet(*WORKED[:1], WORKED[1] % 4))
    rep = E.ReplicatedIndex(*orc.replicate_by_label(Hoods(WORKED[0], WORKED[1] % 4), 2))
    m = ctx.min_label_energies(rep, [1, 4, 2, 9, 0, 5, 3, 8, 6, 2, 7, 5, 1, 9], 7)
    assert m.energy.tolist() == [0, 4, 2, 8, 5, 1, 7] and m.label.tolist() == [1, 0, 0, 1, 1, 1, 0]
    rng = np.random.default_rng(53)
    for _ in range(20):
        g = random_graph(rng, int(rng.integers(2, 30)), 0.25)
        from paper_1809_05018_b200 import inputs
        cl = inputs.maximal_cliques(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
        h, _ = orc.build_neighborhoods(g, cl.offsets, cl.members)
        ctx.set_graph(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
        ctx.set_hoods(E.NeighborhoodSet(h.offsets, h.members))
        M = int(rng.integers(2, 5))
        labels = rng.integers(0, M, g.num_vertices).astype(np.uint32)
        assert np.array_equal(ctx.discord_counts(labels, M), orc.discord_counts(g, labels, M))
        rep = ctx.replicate_by_label(M)
        rep_o = orc.replicate_by_label(h, M)
        assert all(np.array_equal(a, b) for a, b in zip((rep.test_label, rep.old_index, rep.hood_id), rep_o))
        mu, sg = rng.uniform(0, 255, M), rng.uniform(0.5, 60, M)
        e_d = ctx.compute_energies(rep, E.LabelParams(mu, sg), labels, 1.7)
        e_o = orc.compute_energies(g, h, rep_o, mu, sg, labels, 1.7)
        assert np.array_equal(e_d.view(np.uint64), e_o.view(np.uint64))
        coarse = rng.integers(0, 7, len(e_d)).astype(np.float64)  # plenty of ties
        coarse[rng.random(len(coarse)) < 0.05] = np.nan
        coarse[rng.random(len(coarse)) < 0.05] = -0.0
        md = ctx.min_label_energies(rep, coarse, len(h.members))
        me, ml = orc.min_label_energies(rep_o, coarse, len(h.members))
        assert np.array_equal(md.energy.view(np.uint64), me.view(np.uint64))
        assert np.array_equal(md.label, ml)
        argmin = rng.integers(0, M, len(h.members)).astype(np.uint32)
        old = rng.integers(0, M, g.num_vertices).astype(np.uint32)
        assert np.array_equal(ctx.update_labels(argmin, old), orc.update_labels(h, argmin, old))
        slot_hood = ctx.slot_hood_map()
        mins = rng.uniform(0, 100, len(h.members))
        assert np.array_equal(ctx.neighborhood_energy_sums(slot_hood, mins),
                              orc.neighborhood_energy_sums(slot_hood, mins))
        pm, ps = rng.uniform(0, 255, M), rng.uniform(1, 50, M)
        p = ctx.update_parameters(labels, E.LabelParams(pm, ps))
        om, os_ = orc.update_parameters(g.region_mean, labels, pm, ps)
        assert np.array_equal(p.mu, om) and np.array_equal(p.sigma, os_)


def test_fold_topology_long_runs(ctx, orc):
    rng = np.random.default_rng(5)
    keys, vals = [], []
    for h, n in enumerate([1, 3, 1024, 1025, 5000, 2049, 7]):
        keys += [h] * n
        vals += list(rng.uniform(-1e6, 1e6, n) * 10.0 ** rng.integers(-6, 6, n))
    assert np.array_equal(ctx.neighborhood_energy_sums(keys, vals),
                          orc.neighborhood_energy_sums(keys, vals))
    # update_parameters with > 1024 vertices per label: leaf + tree folds
    R = 20000
    g = graph_from_edges(R, [], rng.uniform(0, 255, R) / 7.0)
    ctx.set_graph(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
    for M in (1, 2, 5):
        labels = rng.integers(0, M, R).astype(np.uint32)
        p = ctx.update_parameters(labels, E.LabelParams(np.zeros(M), np.ones(M)))
        om, os_ = orc.update_parameters(g.region_mean, labels, np.zeros(M), np.ones(M))
        assert np.array_equal(p.mu, om) and np.array_equal(p.sigma, os_)
    # empty labels between and after populated ones keep their parameters
    # (engine.cpp:198-213) and must not disturb their neighbors' folds
    for used in ([0, 1, 3], [3], [1, 4], [0]):
        labels = rng.choice(np.array(used, np.uint32), R)
        prev = E.LabelParams(np.arange(5, dtype=np.float64) + 0.5, np.arange(5, dtype=np.float64) + 2)
        p = ctx.update_parameters(labels, prev)
        om, os_ = orc.update_parameters(g.region_mean, labels, prev.mu, prev.sigma)
        assert np.array_equal(p.mu, om) and np.array_equal(p.sigma, os_), used


def test_convergence_and_params_golden(ctx):  # mrf_engine_test.cpp:344-417
    assert ctx.check_convergence([[5.0]] * 4, 3, 1e-4).tolist() == [1]
    assert ctx.check_convergence([[5.0], [5.1], [5.0], [5.0]], 3, 1e-4).tolist() == [0]
    assert ctx.check_convergence([[5.0], [5.0]], 3, 1e-4).tolist() == [0]
    hist = [[1.0, 10.0], [1.0, 20.0], [1.0, 30.0], [1.0, 30.00001]]
    assert ctx.check_convergence(hist, 3, 1e-4).tolist() == [1, 0]
    assert ctx.check_convergence(hist, 1, 1e-4).tolist() == [1, 1]
    g = graph_from_edges(3, [], [10.0, 20.0, 99.0])
    ctx.set_graph(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
    p = ctx.update_parameters([0, 0, 1], E.LabelParams(np.zeros(2), np.ones(2)))
    assert p.mu.tolist() == [15.0, 99.0] and p.sigma.tolist() == [5.0, 1e-3]
    g = graph_from_edges(2, [], [40.0, 60.0])
    ctx.set_graph(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
    p = ctx.update_parameters([0, 0], E.LabelParams(np.array([1.0, 123.5]), np.array([2.0, 4.5])))
    assert p.mu.tolist() == [50.0, 123.5] and p.sigma.tolist() == [10.0, 4.5]
    ctx.set_hoods(E.NeighborhoodSet(*WORKED))
    assert ctx.update_labels([0, 0, 1, 1, 1, 0, 0], [1] * 6).tolist() == [0, 0, 1, 0, 0, 1]


@pytest.mark.parametrize("R,frac0", [(9_000_000, 0.97), (20_000_000, 0.5), (3_000_000, 0.0)])
def test_update_parameters_long_series(orc, R, frac0):
    """Series of > 8200 leaves (> 8.4M elements) take the chunked tree in the
    leaf-fold tail (aligned 1024-partial chunks, then the roots); labels of
    one class only leave the other label empty (keeps its parameters)."""
    rng = np.random.default_rng(R)
    mean = rng.random(R) * 255.0
    labels = (rng.random(R) >= frac0).astype(np.uint32)
    c = E.Context(0)
    try:
        c.set_graph(E.RegionGraph(np.zeros(R + 1, np.uint32), np.zeros(0, np.uint32), mean))
        prev = E.LabelParams(np.array([10.0, 20.0]), np.array([3.0, 4.0]))
        got = c.update_parameters(labels, prev)
    finally:
        c.close()
    mu, sg = orc.update_parameters(mean, labels, prev.mu, prev.sigma)
    assert np.array_equal(got.mu, mu) and np.array_equal(got.sigma, sg)


@pytest.mark.parametrize("R,used", [(1_500_000, [1, 3]), (400_000, [0, 4]), (3_000, [2])])
def test_update_parameters_empty_labels_every_fold_path(orc, R, used):
    """M = 5 with only some labels populated, on the three fold paths of the
    M-step (R = 1.5 M: the persistent streaming kernel; 400 k: the two-grid
    folds; 3 k: the one-cluster sq pass): the populated labels' mu / sigma
    equal the reference's folds, the empty ones keep their parameters
    (engine.cpp:209-220)."""
    rng = np.random.default_rng(R)
    mean = rng.random(R) * 255.0
    labels = rng.choice(np.array(used, np.uint32), R)
    c = E.Context(0)
    try:
        c.set_graph(E.RegionGraph(np.zeros(R + 1, np.uint32), np.zeros(0, np.uint32), mean))
        prev = E.LabelParams(np.arange(5, dtype=np.float64) + 7.5, np.arange(5, dtype=np.float64) + 1)
        got = c.update_parameters(labels, prev)
    finally:
        c.close()
    mu, sg = orc.update_parameters(mean, labels, prev.mu, prev.sigma)
    assert np.array_equal(got.mu, mu) and np.array_equal(got.sigma, sg)
