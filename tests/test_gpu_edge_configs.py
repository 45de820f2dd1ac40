"""Edge configurations through every EM-loop variant: the device-resident loop
with the merged EM tail (default), the device loop without it (full trace),
and the host-log loop (one sync per EM) must agree bit for bit, and with the
oracle, for em_max 0/1, map_max 1/2, window 1, one label (multilabel),
eight labels, beta 0, tiny / huge tolerances."""
import numpy as np
import pytest

from oracle import Config, Graph, Hoods

pytestmark = pytest.mark.gpu
E = pytest.importorskip("paper_1809_05018_b200.engine")
from paper_1809_05018_b200 import inputs  # noqa: E402


@pytest.fixture(scope="module")
def slice_ctx():
    sl = inputs.synthetic_slice(320, 8, seed=23)
    c = E.Context(0)
    c.set_graph(sl.graph)
    c.build_neighborhoods(sl.cliques)
    yield sl, c, c.get_hoods()
    c.close()


CASES = [
    dict(em_max_iters=0),
    dict(em_max_iters=1),
    dict(em_max_iters=6, map_max_iters=1, convergence_window=0),
    dict(em_max_iters=6, map_max_iters=2, convergence_window=1),
    dict(em_max_iters=8, convergence_window=1),
    dict(em_max_iters=8, beta=0.0),
    dict(em_max_iters=8, convergence_tol=1e-12),
    dict(em_max_iters=8, convergence_tol=1e6),
    dict(num_labels=1, em_max_iters=5),
    dict(num_labels=8, em_max_iters=5),
    dict(num_labels=3, em_max_iters=7, map_max_iters=5, convergence_window=2),
]


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
@pytest.mark.parametrize("fixed", [False, True])
def test_em_loop_variants_agree(slice_ctx, orc, case, fixed):
    sl, ctx, hd = slice_ctx
    if case.get("convergence_window", 3) == 0:
        with pytest.raises(E.InputError):  # validate_config: 1 <= L < map_max
            ctx.optimize(E.OptimizerConfig(rng_seed=23, **case))
        return
    cfg = E.OptimizerConfig(rng_seed=23, **case)
    ml = cfg.num_labels != 2
    a = ctx.optimize(cfg, fixed_work=fixed, multilabel=ml, trace_level=E.TRACE_EM)
    b = ctx.optimize(cfg, fixed_work=fixed, multilabel=ml, trace_level=E.TRACE_FULL)
    c = ctx.optimize(cfg, fixed_work=fixed, multilabel=ml, trace_level=E.TRACE_EM, host_log=True)
    for r in (b, c):
        assert np.array_equal(a.labels, r.labels)
        assert np.array_equal(a.mu, r.mu) and np.array_equal(a.sigma, r.sigma)
        assert [e.total_energy for e in a.trace] == [e.total_energy for e in r.trace]
        assert [e.num_map_iters for e in a.trace] == [e.num_map_iters for e in r.trace]
    want = orc.optimize(Graph(sl.graph.offsets, sl.graph.neighbors, sl.graph.region_mean),
                        Hoods(hd.offsets, hd.members),
                        Config(rng_seed=23, **case), fixed_work=fixed, allow_multilabel=ml,
                        full_trace=False)
    assert np.array_equal(a.labels, want.labels)
    assert np.array_equal(a.mu, want.mu) and np.array_equal(a.sigma, want.sigma)
