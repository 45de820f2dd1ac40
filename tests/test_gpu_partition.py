"""Vertex-range partitioned optimize (csrc/partition.cu) on one B200.

A local group runs every partition's vertex / hood passes over its own ranges
with private label, minima, history and counter buffers, moving halos by
device copies -- the exact schedule of the NCCL group.  Results must equal
the one-device optimize (itself pinned to the oracle) bit for bit.
"""
import numpy as np
import pytest

from oracle import C, Config, Graph, Hoods

pytestmark = pytest.mark.gpu
E = pytest.importorskip("paper_1809_05018_b200.engine")
from paper_1809_05018_b200 import inputs  # noqa: E402
from paper_1809_05018_b200.parallel import halo_windows  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = E.Context(0)
    yield c
    c.close()


def _load(ctx, size, block, brick=False, seed=11):
    sl = inputs.synthetic_slice(size, block, brick=brick, seed=seed)
    ctx.set_graph(sl.graph)
    ctx.build_neighborhoods(sl.cliques)
    return sl, ctx.get_hoods()


def _same(a, b):
    assert np.array_equal(a.labels, b.labels)
    assert np.array_equal(a.params.mu, b.params.mu)
    assert np.array_equal(a.params.sigma, b.params.sigma)
    assert [e.total_energy for e in a.trace] == [e.total_energy for e in b.trace]
    assert [e.num_map_iters for e in a.trace] == [e.num_map_iters for e in b.trace]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 7])
@pytest.mark.parametrize("fixed", [False, True])
def test_local_group_matches_one_device(ctx, world, fixed):
    _load(ctx, 1024, 8)  # 128 x 128 regions
    cfg = E.OptimizerConfig(em_max_iters=8, rng_seed=3)
    want = ctx.optimize(cfg, fixed_work=fixed, trace_level=E.TRACE_EM)
    g = E.PartitionGroup.local(ctx, world)
    got = g.optimize(cfg, fixed_work=fixed)
    _same(got, want)
    assert got.stats["em_iters"] == want.stats["em_iters"]
    g.close()


def test_local_group_matches_oracle_and_paths(ctx):
    sl, hd = _load(ctx, 768, 8, seed=5)
    cfg = E.OptimizerConfig(em_max_iters=6, rng_seed=5)
    want = C().optimize(Graph(sl.graph.offsets, sl.graph.neighbors, sl.graph.region_mean),
                        Hoods(hd.offsets, hd.members), Config(rng_seed=5, em_max_iters=6),
                        full_trace=False)
    g = E.PartitionGroup.local(ctx, 3)
    for kw in ({}, {"host_log": True}, {"graphs": False}, {"csr": True}):
        got = g.optimize(cfg, **kw)
        assert np.array_equal(got.labels, want.labels), kw
        assert np.array_equal(got.params.mu, want.mu), kw
        assert np.array_equal(got.params.sigma, want.sigma), kw
        assert [e.total_energy for e in got.trace] == [e.total_energy for e in want.trace], kw
    g.close()


def test_local_group_brick_multilabel(ctx):
    _load(ctx, 1024, 8, brick=True, seed=9)
    cfg = E.OptimizerConfig(num_labels=5, em_max_iters=5, rng_seed=9)
    want = ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_EM, multilabel=True)
    g = E.PartitionGroup.local(ctx, 4)
    _same(g.optimize(cfg, fixed_work=True, multilabel=True), want)
    g.close()


def test_plan_matches_host_mirror(ctx):
    sl, hd = _load(ctx, 1024, 8)
    for world in (2, 3, 5):
        g = E.PartitionGroup.local(ctx, world)
        info = g.info()
        p = halo_windows(sl.graph.offsets, sl.graph.neighbors, hd.offsets, hd.members, world)
        assert info["world"] == world and info["rank"] == -1
        assert (info["vertex_begin"], info["vertex_end"]) == (p.vb[0], p.vb[1])
        assert (info["series_begin"], info["series_end"]) == (p.hb[0], p.hb[1])
        assert info["halo_bytes_per_map"] == p.halo_bytes()
        g.close()


def test_larger_slice_partitions(ctx):
    # 4096^2 block 7: 585 x 585 regions, D's structure at 1/16 scale
    _load(ctx, 4096, 7, seed=42)
    cfg = E.OptimizerConfig(em_max_iters=4, rng_seed=42)
    want = ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_EM)
    for world in (2, 8):
        g = E.PartitionGroup.local(ctx, world)
        _same(g.optimize(cfg, fixed_work=True), want)
        g.close()


def test_partition_errors(ctx):
    _load(ctx, 512, 8)
    g = E.PartitionGroup.local(ctx, 2)
    with pytest.raises(ValueError):  # the per-MAP trace is one-device only
        g.optimize(E.OptimizerConfig(em_max_iters=2), trace_level=E.TRACE_FULL)
    with pytest.raises(E.InputError):
        g.optimize(E.OptimizerConfig(num_labels=3), multilabel=False)
    g.close()
    with pytest.raises(ValueError):
        E.PartitionGroup.local(ctx, 0)
    with pytest.raises(ValueError):
        E.PartitionGroup.local(ctx, 65)


def test_nccl_single_rank_group(ctx):
    """NCCL is loaded at run time; a world-1 communicator runs the same path."""
    _load(ctx, 512, 8)
    cfg = E.OptimizerConfig(em_max_iters=4, rng_seed=1)
    want = ctx.optimize(cfg, trace_level=E.TRACE_EM)
    uid = E.nccl_unique_id()
    assert len(uid) == 128
    g = E.PartitionGroup.nccl(ctx, uid, 0, 1)
    _same(g.optimize(cfg), want)
    g.close()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_local_group_split_hood_pass(ctx, world, monkeypatch):
    """DPMRF_GROUP_SPLIT=1: the schedule of NCCL groups -- halo exchange on a
    side stream while the interior hoods are folded, boundary hoods after --
    on the local transport; results equal the one-device run bit for bit."""
    _load(ctx, 1024, 8, seed=13)
    cfg = E.OptimizerConfig(em_max_iters=6, rng_seed=13)
    for fixed in (False, True):
        want = ctx.optimize(cfg, fixed_work=fixed, trace_level=E.TRACE_EM)
        monkeypatch.setenv("DPMRF_GROUP_SPLIT", "1")
        g = E.PartitionGroup.local(ctx, world)
        monkeypatch.delenv("DPMRF_GROUP_SPLIT")
        try:
            got = g.optimize(cfg, fixed_work=fixed)
        finally:
            g.close()
        _same(got, want)
