"""CUDA path (through the C ABI) vs the pinned oracle -- run on the B200.

Bar: bit-exact labels, parameters, total energies and per-MAP hood energies /
flags (the reference is bit-deterministic by design, proj/README.md:91-104;
the north_star tolerance -- labels exact where the energy gap > 1e-6
relative, parameters within 1e-5 relative -- is therefore met with margin).
"""
import numpy as np
import pytest

from golden_io import Fixture, names
from oracle import Config, Graph, Hoods, graph_from_edges, random_graph

pytestmark = pytest.mark.gpu

E = pytest.importorskip("paper_1809_05018_b200.engine")


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    c = E.Context(0)
    yield c
    c.close()


def to_cfg(c: Config) -> "E.OptimizerConfig":
    return E.OptimizerConfig(c.num_labels, c.em_max_iters, c.map_max_iters, c.convergence_window,
                             c.convergence_tol, c.beta, c.rng_seed)


def upload(ctx, g: Graph, h: Hoods):
    ctx.set_graph(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
    ctx.set_hoods(E.NeighborhoodSet(h.offsets, h.members))


def same(a, b, full=True):
    assert np.array_equal(np.asarray(a.labels, np.uint32), np.asarray(b.labels, np.uint32))
    assert np.array_equal(a.mu, b.mu) and np.array_equal(a.sigma, b.sigma)
    assert len(a.trace) == len(b.trace)
    for x, y in zip(a.trace, b.trace):
        assert x.total_energy == y.total_energy
        assert bool(x.converged) == bool(y.converged)
        assert x.num_map_iters == y.num_map_iters
        assert np.array_equal(x.mu, y.mu) and np.array_equal(x.sigma, y.sigma)
        if full:
            assert len(x.map_iters) == len(y.map_iters)
            for m, n in zip(x.map_iters, y.map_iters):
                assert np.array_equal(m.hood_energy.view(np.uint64), n.hood_energy.view(np.uint64))
                assert np.array_equal(m.converged, n.converged)


# ---- committed reference fixtures (configs A, acceptance 128^2, block 7, M=5 brick) ----
@pytest.mark.parametrize("name", names())
def test_fixture_optimize(ctx, name):
    f = Fixture(name)
    upload(ctx, f.graph, f.hoods)
    r = ctx.optimize(to_cfg(f.cfg), fixed_work=f.fixed, multilabel=f.multilabel)
    f.check(r)


@pytest.mark.parametrize("layout", ["packed", "unfused", "csr"])
@pytest.mark.parametrize("graphs", [False, True])
def test_execution_modes_agree(ctx, graphs, layout):
    # fused MAP-boundary launches vs two kernels per MAP iteration, each with
    # and without CUDA-graph replay, over the packed delta layout and the u32
    # CSR: identical results and full traces (device loop and host-log loop)
    for name in ("configA_256_grid8", "m5_128_brick8", "configA_252_grid7"):
        f = Fixture(name)
        upload(ctx, f.graph, f.hoods)
        for host_log in (False, True):
            r = ctx.optimize(to_cfg(f.cfg), fixed_work=f.fixed, multilabel=f.multilabel,
                             graphs=graphs, csr=layout == "csr", fused=layout != "unfused",
                             host_log=host_log)
            f.check(r)
            assert r.stats["graphs"] == (1 if graphs else 0)
        for level in (E.TRACE_NONE, E.TRACE_EM):
            for timing in (False, True):  # timing forces the host-log loop
                r2 = ctx.optimize(to_cfg(f.cfg), fixed_work=f.fixed, multilabel=f.multilabel,
                                  graphs=graphs, trace_level=level, kernel_timing=timing,
                                  csr=layout == "csr", fused=layout != "unfused")
                assert np.array_equal(r2.labels, r.labels) and np.array_equal(r2.mu, r.mu)
                assert np.array_equal(r2.sigma, r.sigma)


@pytest.mark.parametrize("name", names())
def test_fixture_build_neighborhoods(ctx, name):
    f = Fixture(name)
    ctx.set_graph(E.RegionGraph(f.graph.offsets, f.graph.neighbors, f.graph.region_mean))
    n = ctx.build_neighborhoods(E.CliqueSet(*f.cliques))
    h = ctx.get_hoods()
    assert n == len(f.hoods.members)
    assert np.array_equal(h.offsets, f.hoods.offsets)
    assert np.array_equal(h.members, f.hoods.members)
    assert np.array_equal(h.source_clique, np.arange(len(h.offsets) - 1, dtype=np.uint32))
    # the device-built hoods drive optimize to the same fixture
    r = ctx.optimize(to_cfg(f.cfg), fixed_work=f.fixed, multilabel=f.multilabel)
    f.check(r)


# ---- random instances vs the C restatement ------------------------------------------
def test_random_graphs_vs_oracle(ctx, orc):
    rng = np.random.default_rng(7)
    for i in range(60):
        n = int(rng.integers(1, 60))
        g = random_graph(rng, n, float(rng.uniform(0.02, 0.7)))
        # cliques from the product's host builder, hoods from the device
        from paper_1809_05018_b200 import inputs
        cl = inputs.maximal_cliques(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
        h, _ = orc.build_neighborhoods(g, cl.offsets, cl.members)
        ctx.set_graph(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
        ctx.build_neighborhoods(cl)
        hd = ctx.get_hoods()
        assert np.array_equal(hd.offsets, h.offsets) and np.array_equal(hd.members, h.members)
        M = int(rng.choice([2, 2, 3, 5]))
        cfg = Config(num_labels=M, rng_seed=int(rng.integers(0, 2**62)),
                     beta=float(rng.uniform(0, 3)), em_max_iters=int(rng.integers(0, 8)),
                     map_max_iters=int(rng.integers(2, 8)))
        cfg.convergence_window = int(rng.integers(1, cfg.map_max_iters))
        for fixed in (False, True):
            a = orc.optimize(g, h, cfg, fixed_work=fixed, allow_multilabel=True)
            b = ctx.optimize(to_cfg(cfg), fixed_work=fixed, multilabel=True)
            same(a, b)


def test_handmade_hoods_empty_and_uncovered(ctx, orc):
    # hoods that skip vertices and include empty hoods (reduce_by_key runs,
    # engine.cpp:150) -- never produced by build_neighborhoods, allowed by the API
    g = graph_from_edges(6, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5)],
                         [10.0, 200.0, 15.0, 190.0, 30.0, 60.0])
    h = Hoods(np.array([0, 3, 3, 5, 5], np.uint32), np.array([0, 1, 2, 2, 3], np.uint32))
    upload(ctx, g, h)
    for seed in range(5):
        cfg = Config(rng_seed=seed, em_max_iters=6)
        same(orc.optimize(g, h, cfg), ctx.optimize(to_cfg(cfg)))
        same(orc.optimize(g, h, cfg, fixed_work=True), ctx.optimize(to_cfg(cfg), fixed_work=True))


def test_handmade_hoods_out_of_order(ctx, orc):
    # members not ascending (the API allows any order; the sum folds in slot
    # order): the delta-packed hood layout must not be used for them
    rng = np.random.default_rng(11)
    n = 40
    g = graph_from_edges(n, [(v, v + 1) for v in range(n - 1)], rng.uniform(0, 255, n))
    mem, off = [], [0]
    for v in range(n):
        m = [v] + [u for u in (v - 1, v + 1) if 0 <= u < n]
        rng.shuffle(m)
        mem += m
        off.append(len(mem))
    h = Hoods(np.array(off, np.uint32), np.array(mem, np.uint32))
    upload(ctx, g, h)
    for seed in range(4):
        cfg = Config(rng_seed=seed, em_max_iters=5)
        same(orc.optimize(g, h, cfg), ctx.optimize(to_cfg(cfg)))
        same(orc.optimize(g, h, cfg, fixed_work=True), ctx.optimize(to_cfg(cfg), fixed_work=True))


def test_large_hood_leaf_tree_fold(ctx, orc):
    # a star hub with > 1024 neighbors: hood sums switch to the leaf/tree fold
    n = 2600
    rng = np.random.default_rng(3)
    g = graph_from_edges(n, [(0, v) for v in range(1, n)], rng.uniform(0, 255, n) / 7.0)
    from paper_1809_05018_b200 import inputs
    cl = inputs.maximal_cliques(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
    h, _ = orc.build_neighborhoods(g, cl.offsets, cl.members)
    assert int(np.diff(h.offsets).max()) > 1024
    ctx.set_graph(E.RegionGraph(g.offsets, g.neighbors, g.region_mean))
    ctx.build_neighborhoods(cl)  # exercises the > 1024-candidate block sort
    hd = ctx.get_hoods()
    assert np.array_equal(hd.offsets, h.offsets) and np.array_equal(hd.members, h.members)
    cfg = Config(rng_seed=9, em_max_iters=4)
    same(orc.optimize(g, h, cfg, fixed_work=True), ctx.optimize(to_cfg(cfg), fixed_work=True))


@pytest.mark.parametrize("size,block,brick,M", [(512, 8, False, 2), (384, 7, False, 2),
                                                (512, 8, True, 5), (320, 6, True, 3)])
def test_phantom_fixed_work_vs_oracle(ctx, orc, size, block, brick, M):
    from paper_1809_05018_b200 import inputs
    sl = inputs.synthetic_slice(size, block, brick=brick, seed=11)
    g = Graph(sl.graph.offsets, sl.graph.neighbors, sl.graph.region_mean)
    ctx.set_graph(sl.graph)
    ctx.build_neighborhoods(sl.cliques)
    hd = ctx.get_hoods()
    h = Hoods(hd.offsets, hd.members)
    cfg = Config(num_labels=M, rng_seed=5, em_max_iters=5)
    same(orc.optimize(g, h, cfg, fixed_work=True, allow_multilabel=True),
         ctx.optimize(to_cfg(cfg), fixed_work=True, multilabel=True))
    if M == 2:
        same(orc.optimize(g, h, Config(rng_seed=5)), ctx.optimize(to_cfg(Config(rng_seed=5))))


def test_large_graph_grouping_path_vs_oracle(ctx, orc):
    """tiles x labels > kSelfScanMax (8192) takes the large-graph grouping
    (k_tile_chunks / k_tile_offsets / k_label_scatter_warp, one warp per
    256-vertex tile) that otherwise only the 16384^2 bench shape reaches:
    1024^2 block 4 (65 536 regions, 256 tiles) with 40 labels."""
    from paper_1809_05018_b200 import inputs
    sl = inputs.synthetic_slice(1024, 4, seed=3)
    g = Graph(sl.graph.offsets, sl.graph.neighbors, sl.graph.region_mean)
    ctx.set_graph(sl.graph)
    ctx.build_neighborhoods(sl.cliques)
    hd = ctx.get_hoods()
    h = Hoods(hd.offsets, hd.members)
    assert (len(g.offsets) - 1 + 255) // 256 * 40 > 8192
    cfg = Config(num_labels=40, rng_seed=9, em_max_iters=3)
    same(orc.optimize(g, h, cfg, fixed_work=True, allow_multilabel=True),
         ctx.optimize(to_cfg(cfg), fixed_work=True, multilabel=True))


@pytest.mark.parametrize("map_max,window", [(31, 2), (32, 5), (33, 3), (40, 1)])
def test_long_map_loops_vs_oracle(ctx, orc, map_max, window):
    """MAP loops around the warp width: the sum pass reads the per-iteration
    counters one lane each up to 32 iterations, a loop beyond (early exits
    and fixed work)."""
    from paper_1809_05018_b200 import inputs
    sl = inputs.synthetic_slice(256, 8, seed=3)
    g = Graph(sl.graph.offsets, sl.graph.neighbors, sl.graph.region_mean)
    ctx.set_graph(sl.graph)
    ctx.build_neighborhoods(sl.cliques)
    hd = ctx.get_hoods()
    h = Hoods(hd.offsets, hd.members)
    for tol in (1e-6, 1e-300):  # (1e-300: only bit-equal sums converge)
        cfg = Config(rng_seed=8, em_max_iters=4, map_max_iters=map_max, convergence_window=window,
                     convergence_tol=tol)
        for fixed in (False, True):
            same(orc.optimize(g, h, cfg, fixed_work=fixed), ctx.optimize(to_cfg(cfg), fixed_work=fixed))


def test_config_b_against_reference(ctx, ref):
    """Config B shape (2560^2, block 8) vs the reference library itself:
    reference semantics, full trace; and 2 EM of fixed work."""
    from paper_1809_05018_b200 import inputs
    p = ref.phantom(2560, 8, seed=42, threads=4)
    sl = inputs.synthetic_slice(2560, 8, seed=42)
    ctx.set_graph(sl.graph)
    ctx.build_neighborhoods(sl.cliques)
    hd = ctx.get_hoods()
    assert np.array_equal(hd.members, p.hoods().members)
    cfg = Config(rng_seed=42)
    same(p.optimize(cfg, threads=8), ctx.optimize(to_cfg(cfg)))
    cfg2 = Config(rng_seed=42, em_max_iters=2)
    same(p.optimize(cfg2, threads=8, mode=1, fixed_work=True),
         ctx.optimize(to_cfg(cfg2), fixed_work=True))


def test_trace_levels_and_determinism(ctx):
    f = Fixture("configA_256_grid8")
    upload(ctx, f.graph, f.hoods)
    full = ctx.optimize(to_cfg(f.cfg))
    em = ctx.optimize(to_cfg(f.cfg), trace_level=E.TRACE_EM)
    none = ctx.optimize(to_cfg(f.cfg), trace_level=E.TRACE_NONE)
    assert np.array_equal(full.labels, none.labels) and np.array_equal(full.mu, none.mu)
    assert [e.total_energy for e in em.trace] == [e.total_energy for e in full.trace]
    assert none.trace == [] and all(e.map_iters == [] for e in em.trace)
    for _ in range(3):
        again = ctx.optimize(to_cfg(f.cfg))
        same(full, again)


# ---- error convention ---------------------------------------------
def test_errors(ctx):
    g = graph_from_edges(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)], [10, 12, 200, 210])
    h = Hoods(np.array([0, 4], np.uint32), np.array([0, 1, 2, 3], np.uint32))
    upload(ctx, g, h)
    base = E.OptimizerConfig()
    for kw in [dict(num_labels=3), dict(em_max_iters=-1), dict(map_max_iters=0),
               dict(convergence_window=0), dict(convergence_window=10),
               dict(convergence_tol=0.0), dict(beta=-0.5)]:
        cfg = E.OptimizerConfig(**{**base.__dict__, **kw})
        with pytest.raises(E.InputError):
            ctx.optimize(cfg, multilabel=False)
    ctx.optimize(E.OptimizerConfig(beta=0.0))
    with pytest.raises(E.InputError):
        ctx.build_neighborhoods(E.CliqueSet(np.array([0, 4], np.uint32),
                                            np.array([0, 1, 2, 3], np.uint32)), k=2)
    with pytest.raises(IndexError):
        ctx.build_neighborhoods(E.CliqueSet(np.array([0, 1], np.uint32), np.array([9], np.uint32)))
    ctx.set_hoods(E.NeighborhoodSet(np.array([0, 2], np.uint32), np.array([0, 7], np.uint32)))
    with pytest.raises(IndexError):
        ctx.optimize(E.OptimizerConfig())
    # em_max_iters == 0 never touches the hoods (optimize.cpp:35)
    r = ctx.optimize(E.OptimizerConfig(em_max_iters=0, rng_seed=99))
    params, lab = ctx.init_random(2, 4, 99)
    assert np.array_equal(r.labels, lab) and np.array_equal(r.mu, params.mu)
    with pytest.raises(E.InputError):
        ctx.init_random(3, 4, 0)
    with pytest.raises(ValueError):
        ctx.update_parameters([0, 0, 2, 1], E.LabelParams(np.zeros(2), np.ones(2)))


def test_invalid_csr_rejected_by_the_prepare_batch(ctx):
    """prepare() builds the packed layouts and cover flags in the same batch as
    the validation (before the host sees it): non-monotone offsets must still
    come back as the reference's invalid_argument, with the context usable."""
    g = graph_from_edges(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)], [10, 12, 200, 210])
    good = Hoods(np.array([0, 2, 4], np.uint32), np.array([0, 1, 2, 3], np.uint32))
    bad_h = E.NeighborhoodSet(np.array([0, 3, 2, 4], np.uint32), np.array([0, 1, 2, 3], np.uint32))
    for arrays in (False, True):
        upload(ctx, g, good)
        with pytest.raises(ValueError, match="neighborhood offsets"):
            if arrays:
                ctx.optimize_arrays(E.RegionGraph(g.offsets, g.neighbors, g.region_mean), bad_h,
                                    E.OptimizerConfig())
            else:
                ctx.set_hoods(bad_h)
                ctx.optimize(E.OptimizerConfig())
    bad_g = E.RegionGraph(np.array([0, 3, 2, 9, 12], np.uint32), np.asarray(g.neighbors, np.uint32),
                          np.asarray(g.region_mean, np.float64))
    ctx.set_graph(bad_g)
    ctx.set_hoods(E.NeighborhoodSet(good.offsets, good.members))
    with pytest.raises(ValueError, match="region graph offsets"):
        ctx.optimize(E.OptimizerConfig())
    upload(ctx, g, good)  # the context recovers
    ctx.optimize(E.OptimizerConfig(rng_seed=3))


def test_two_vertices_per_thread_path(ctx):
    """R >= 2^20 switches the fused launch to two vertices per thread
    (engine.cu kVertsPerThreadMin); it must equal the unfused two-kernel
    path (one vertex per thread, pinned to the oracle above) bit for bit."""
    from paper_1809_05018_b200 import inputs
    sl = inputs.synthetic_slice(4104, 4, seed=21)  # > 2^20 vertices: also the many-block tile scan
    assert sl.graph.num_vertices >= 1 << 20
    ctx.set_graph(sl.graph)
    ctx.build_neighborhoods(sl.cliques)
    for fixed in (True, False):
        cfg = E.OptimizerConfig(em_max_iters=4, rng_seed=21)
        a = ctx.optimize(cfg, fixed_work=fixed, trace_level=E.TRACE_FULL)
        b = ctx.optimize(cfg, fixed_work=fixed, trace_level=E.TRACE_FULL, fused=False)
        assert np.array_equal(a.labels, b.labels)
        assert np.array_equal(a.mu, b.mu) and np.array_equal(a.sigma, b.sigma)
        assert [e.total_energy for e in a.trace] == [e.total_energy for e in b.trace]
        for ea, eb in zip(a.trace, b.trace):
            assert len(ea.map_iters) == len(eb.map_iters)
            for ma, mb in zip(ea.map_iters, eb.map_iters):
                assert np.array_equal(ma.hood_energy, mb.hood_energy)
                assert np.array_equal(ma.converged, mb.converged)


def test_optimize_arrays_one_call(ctx):
    """dpmrf_optimize_arrays (upload + optimize in one call) == set_graph +
    set_hoods + optimize, including after the context held another graph."""
    from paper_1809_05018_b200 import inputs
    sl = inputs.synthetic_slice(512, 8, seed=17)
    ctx.set_graph(sl.graph)
    ctx.build_neighborhoods(sl.cliques)
    hoods = ctx.get_hoods()
    cfg = E.OptimizerConfig(em_max_iters=6, rng_seed=17)
    want = ctx.optimize(cfg, trace_level=E.TRACE_EM)
    other = inputs.synthetic_slice(256, 8, seed=1)  # replace the resident inputs first
    ctx.set_graph(other.graph)
    ctx.build_neighborhoods(other.cliques)
    got = ctx.optimize_arrays(sl.graph, hoods, cfg, trace_level=E.TRACE_EM)
    assert np.array_equal(got.labels, want.labels)
    assert np.array_equal(got.mu, want.mu) and np.array_equal(got.sigma, want.sigma)
    assert [e.total_energy for e in got.trace] == [e.total_energy for e in want.trace]
    with pytest.raises(ValueError):  # a bad CSR is reported, not run
        bad = E.NeighborhoodSet(np.array([0, 5, 3], np.uint32), hoods.members[:5])
        ctx.optimize_arrays(sl.graph, bad, cfg)


def test_concurrent_calls_on_one_context_serialize(ctx):
    """Entry points hold the context's mutex: two host threads interleaving
    optimize_arrays on ONE context with DIFFERENT graphs each get their own
    result (the reference's pool serializes submissions, backend.cpp:45)."""
    import threading
    from paper_1809_05018_b200 import inputs
    cfg = E.OptimizerConfig(em_max_iters=4, rng_seed=5)
    cases = []
    for n, seed in ((512, 3), (384, 4)):
        sl = inputs.synthetic_slice(n, 8, seed=seed)
        ctx.set_graph(sl.graph)
        ctx.build_neighborhoods(sl.cliques)
        hoods = ctx.get_hoods()
        want = ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_NONE)
        cases.append((sl.graph, hoods, want))
    errors = []

    def worker(graph, hoods, want):
        try:
            for _ in range(6):
                got = ctx.optimize_arrays(graph, hoods, cfg, fixed_work=True,
                                          trace_level=E.TRACE_NONE)
                assert np.array_equal(got.labels, want.labels)
                assert np.array_equal(got.mu, want.mu)
                assert np.array_equal(got.sigma, want.sigma)
        except Exception as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=worker, args=c) for c in cases]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("env,val", [("DPMRF_NO_K12", "1"), ("DPMRF_CLUSTER_SQ", "0")])
def test_opt_in_layouts_agree(env, val, monkeypatch):
    """16-slot rows for brick hoods (DPMRF_NO_K12=1), and the grid-wide sq
    pass with its global-ticket tail instead of the one-cluster sq pass on
    small graphs (DPMRF_CLUSTER_SQ=0), reproduce the fixtures and the
    default path."""
    from paper_1809_05018_b200 import inputs
    monkeypatch.setenv(env, val)
    c = E.Context(0)
    monkeypatch.delenv(env)
    base = E.Context(0)
    try:
        for name in ("configA_256_grid8", "m5_128_brick8", "configA_252_grid7"):
            f = Fixture(name)
            upload(c, f.graph, f.hoods)
            for fixed in (f.fixed, True):
                r = c.optimize(to_cfg(f.cfg), fixed_work=fixed, multilabel=f.multilabel,
                               trace_level=E.TRACE_EM)
                if fixed == f.fixed:
                    f.check(r)
        for size, seed, brick in ((1024, 3, False), (2560, 42, False), (1000, 5, True)):
            sl = inputs.synthetic_slice(size, 8, seed=seed, brick=brick)
            for ctx_ in (c, base):
                ctx_.set_graph(sl.graph)
                ctx_.build_neighborhoods(sl.cliques)
            for fixed in (False, True):
                cfg = E.OptimizerConfig(em_max_iters=8, rng_seed=seed)
                got = c.optimize(cfg, fixed_work=fixed, trace_level=E.TRACE_EM)
                want = base.optimize(cfg, fixed_work=fixed, trace_level=E.TRACE_EM)
                same(got, want, full=False)
    finally:
        c.close()
        base.close()


def test_grids_with_holes_vs_oracle(ctx, orc):
    """Row-major grids with missing edges and handmade hoods (uncovered
    vertices, members up to three rows below and columns -1..3 of the first)
    -- the packed layouts' delta ranges at small strides -- and low-degree
    random graphs with one-member hoods."""
    rng = np.random.default_rng(21)
    layouts = set()
    for i in range(30):
        n = int(rng.integers(2, 80))
        if i % 2:
            g = random_graph(rng, n, float(rng.uniform(0.01, 0.06)))
            h = Hoods(np.arange(n + 1, dtype=np.uint32), np.arange(n, dtype=np.uint32))
        else:
            W = int(rng.integers(2, 9))
            n = W * int(rng.integers(1, 9))
            edges = [(v, v + 1) for v in range(n) if (v + 1) % W and v + 1 < n and rng.random() < 0.8]
            edges += [(v, v + W) for v in range(n - W) if rng.random() < 0.8]
            g = graph_from_edges(n, edges, rng.uniform(0, 255, n))
            off, mem = [0], []
            for v in range(n):
                if rng.random() < 0.15:
                    continue
                cand = (v + 1, v + 3, v + W, v + W + 1, v + 2 * W - 1, v + 3 * W + 2)
                m = sorted({v} | {u for u in cand if u < n and rng.random() < 0.6})
                mem += m
                off.append(len(mem))
            h = Hoods(np.array(off, np.uint32), np.array(mem, np.uint32))
        upload(ctx, g, h)
        cfg = Config(rng_seed=int(rng.integers(0, 2**62)), em_max_iters=int(rng.integers(1, 6)),
                     beta=float(rng.uniform(0, 3)))
        for fixed in (False, True):
            r = ctx.optimize(to_cfg(cfg), fixed_work=fixed)
            same(orc.optimize(g, h, cfg, fixed_work=fixed), r)
            layouts.add(r.stats["packed_layout"])
    assert 408 in layouts


@pytest.mark.parametrize("size,brick,M", [(4096, False, 2), (4096, True, 3)])
def test_stream_fold_matches_two_pass(size, brick, M, monkeypatch):
    """Many-leaf graphs (> 4 x 148 leaves): the persistent streaming M-step
    (k_mstep_stream: quarter-leaf ring per chain, chunk/series tickets, grid
    barrier between the passes, label move-back on odd MAP counts) equals the
    two-pass folds (DPMRF_STREAM=0) bit for bit, with and without early exits,
    over the EM trace."""
    from paper_1809_05018_b200 import inputs
    monkeypatch.setenv("DPMRF_STREAM", "0")
    two = E.Context(0)
    monkeypatch.delenv("DPMRF_STREAM")
    one = E.Context(0)
    try:
        sl = inputs.synthetic_slice(size, 8, seed=21, brick=brick)
        for c in (one, two):
            c.set_graph(sl.graph)
            c.build_neighborhoods(sl.cliques)
        for fixed in (False, True):
            cfg = E.OptimizerConfig(num_labels=M, em_max_iters=7, rng_seed=21)
            got = one.optimize(cfg, fixed_work=fixed, multilabel=M != 2, trace_level=E.TRACE_EM)
            want = two.optimize(cfg, fixed_work=fixed, multilabel=M != 2, trace_level=E.TRACE_EM)
            same(got, want, full=False)
            assert got.stats["kernel_launches"] < want.stats["kernel_launches"]
    finally:
        one.close()
        two.close()


@pytest.mark.parametrize("size,block,brick,M,seed", [
    (512, 8, False, 2, 3), (1000, 8, False, 2, 9), (768, 8, True, 5, 4), (2560, 8, False, 2, 42),
    (4096, 8, False, 2, 21), (2304, 7, False, 2, 8), (2560, 8, True, 5, 42)])
def test_active_set_matches_dense(ctx, size, block, brick, M, seed):
    """active_set=True (extension, DPMRF_RUN_ACTIVE_SET): vertices re-evaluated
    only when a neighbor's label (or their own label / minimum) changed,
    series folded only when a member's minimum changed or their window is
    open -- the labels, parameters and every EM record (total energy, MAP
    count, converged flag) equal the dense run's bit for bit, with and
    without early exits."""
    from paper_1809_05018_b200 import inputs
    sl = inputs.synthetic_slice(size, block, brick=brick, seed=seed)
    ctx.set_graph(sl.graph)
    ctx.build_neighborhoods(sl.cliques)
    for fixed in (False, True):
        cfg = E.OptimizerConfig(num_labels=M, em_max_iters=8, rng_seed=seed)
        want = ctx.optimize(cfg, fixed_work=fixed, multilabel=M != 2, trace_level=E.TRACE_EM)
        got = ctx.optimize(cfg, fixed_work=fixed, multilabel=M != 2, trace_level=E.TRACE_EM,
                           active_set=True)
        # (grid graphs with two labels; brick graphs keep the dense loop)
        assert got.stats["active_set"] == (0 if brick else 1)
        same(got, want, full=False)
        assert got.stats["map_iters_total"] == want.stats["map_iters_total"]
    # a full trace falls back to the dense loop (every row is needed)
    r = ctx.optimize(E.OptimizerConfig(num_labels=M, em_max_iters=2, rng_seed=seed),
                     multilabel=M != 2, trace_level=E.TRACE_FULL, active_set=True)
    assert r.stats["active_set"] == 0
