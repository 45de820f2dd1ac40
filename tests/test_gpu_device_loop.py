"""The device-resident EM loop: log(sigma) evaluated on the device (correctly
rounded, double-double) and verified against the host libm afterwards.

* the device log is correctly rounded (checked against Python's Decimal);
* it equals the host libm's log wherever the latter is correctly rounded;
* device-loop and host-log runs of optimize() agree bit for bit, including
  the per-EM trace, under reference semantics and fixed work.
"""
import math
import random
from decimal import Decimal, getcontext

import numpy as np
import pytest

from golden_io import Fixture, names

pytestmark = pytest.mark.gpu
E = pytest.importorskip("paper_1809_05018_b200.engine")


@pytest.fixture(scope="module")
def ctx():
    c = E.Context(0)
    yield c
    c.close()


def cr_log(x):
    getcontext().prec = 60
    return float(Decimal(x).ln())  # Decimal -> float rounds correctly


def test_device_log_is_correctly_rounded(ctx):
    rnd = random.Random(17)
    xs = [1.0, 2.0, 0.5, 1e-3, 255.0, math.e, 1.0 + 2.0 ** -52, 1.0 - 2.0 ** -53, 0.7071067811865476,
          1.4142135623730951, float.fromhex("0x1.d9f8ce3f7c27ep-1"),
          float.fromhex("0x1.400112ac2c1aap+0")]
    xs += [rnd.uniform(1e-3, 255.0) for _ in range(3000)]
    xs += [math.exp(rnd.uniform(-7.0, 5.6)) for _ in range(3000)]
    xs += [rnd.uniform(0.6, 1.6) for _ in range(2000)]
    got = ctx.debug_log(xs)
    want = np.array([cr_log(x) for x in xs])
    bad = np.nonzero(got != want)[0]
    assert len(bad) == 0, [(xs[i].hex(), got[i].hex(), want[i].hex()) for i in bad[:5]]
    host = np.array([math.log(x) for x in xs])
    agree = np.mean(host == got)
    assert agree > 0.99  # glibc's log is correctly rounded almost everywhere


@pytest.mark.parametrize("name", names())
def test_device_loop_matches_host_log_loop(ctx, name):
    f = Fixture(name)
    ctx.set_graph(E.RegionGraph(f.graph.offsets, f.graph.neighbors, f.graph.region_mean))
    ctx.set_hoods(E.NeighborhoodSet(f.hoods.offsets, f.hoods.members))
    cfg = E.OptimizerConfig(f.cfg.num_labels, f.cfg.em_max_iters, f.cfg.map_max_iters,
                            f.cfg.convergence_window, f.cfg.convergence_tol, f.cfg.beta,
                            f.cfg.rng_seed)
    for level in (E.TRACE_EM, E.TRACE_FULL):
        dev = ctx.optimize(cfg, fixed_work=f.fixed, trace_level=level, multilabel=f.multilabel)
        host = ctx.optimize(cfg, fixed_work=f.fixed, trace_level=level, multilabel=f.multilabel,
                            host_log=True)
        assert dev.stats["device_loop"] == 1 or dev.stats["device_log_fallbacks"] >= 1
        assert host.stats["device_loop"] == 0
        assert np.array_equal(dev.labels, host.labels)
        assert np.array_equal(dev.mu, host.mu) and np.array_equal(dev.sigma, host.sigma)
        assert [(e.total_energy, e.converged, e.num_map_iters) for e in dev.trace] == \
               [(e.total_energy, e.converged, e.num_map_iters) for e in host.trace]
        f.check(dev, exact_trace=level == E.TRACE_FULL)
        if level == E.TRACE_FULL:  # every MAP row of every EM equal to the host-log loop's
            for a, b in zip(dev.trace, host.trace):
                assert len(a.map_iters) == len(b.map_iters) == a.num_map_iters
                for m, n in zip(a.map_iters, b.map_iters):
                    assert np.array_equal(m.hood_energy.view(np.uint64),
                                          n.hood_energy.view(np.uint64))
                    assert np.array_equal(m.converged, n.converged)


def test_device_loop_long_runs(ctx, orc):
    # 2560^2 would take the oracle ~7 s per EM; use 768^2 with 12 EM of fixed work
    from oracle import Config, Graph, Hoods
    from paper_1809_05018_b200 import inputs
    sl = inputs.synthetic_slice(768, 8, seed=123)
    ctx.set_graph(sl.graph)
    ctx.build_neighborhoods(sl.cliques)
    hd = ctx.get_hoods()
    cfg = E.OptimizerConfig(em_max_iters=12, rng_seed=123)
    dev = ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_EM)
    want = orc.optimize(Graph(sl.graph.offsets, sl.graph.neighbors, sl.graph.region_mean),
                        Hoods(hd.offsets, hd.members), Config(em_max_iters=12, rng_seed=123),
                        fixed_work=True, full_trace=False)
    assert np.array_equal(dev.labels, want.labels)
    assert np.array_equal(dev.mu, want.mu) and np.array_equal(dev.sigma, want.sigma)
    assert [e.total_energy for e in dev.trace] == [e.total_energy for e in want.trace]
    assert dev.stats["device_loop"] == 1 or dev.stats["device_log_fallbacks"] >= 1
