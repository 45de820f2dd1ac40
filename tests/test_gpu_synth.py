"""Synthetic inputs on the device (csrc/synth.cu) vs the host builder and the
reference: gen_phantom + corrupt (phantom.cpp:54-150) bit for bit, grid and
brick oversegmentations, and the fully device-resident pipeline
(phantom -> ... -> neighborhoods -> optimize) vs the host-input pipeline."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
E = pytest.importorskip("paper_1809_05018_b200.engine")
from paper_1809_05018_b200 import inputs  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = E.Context(0)
    yield c
    c.close()


SPECS = [  # (w, h, pore, sp, gauss, ringing, seed)
    (256, 256, 0.25, 0.05, 100.0, True, 42),
    (300, 170, 0.4, 0.0, 0.0, False, 7),
    (97, 61, 0.1, 0.2, 30.0, False, 3),
    (512, 512, 0.25, 0.0, 0.0, True, 11),
    (2560, 2560, 0.25, 0.05, 100.0, True, 42),  # config B's image
]


@pytest.mark.parametrize("spec", SPECS)
def test_phantom_matches_host_builder(ctx, spec):
    w, h, pore, sp, gauss, ring, seed = spec
    truth, image, ties = ctx.make_phantom(w, h, pore, sp, gauss, ring, seed)
    ps = inputs.PhantomSpec(w, h, pore, sp, gauss, ring, seed)
    t_host, clean = inputs.gen_phantom(ps)
    assert np.array_equal(truth, t_host)
    assert np.array_equal(image, inputs.corrupt(clean, ps))
    assert ties <= 8  # rounding ties resolved with glibc are rare


def test_phantom_matches_reference(ctx, ref):
    truth, image, _ = ctx.make_phantom(256, 192, 0.25, 0.05, 100.0, True, 5)
    px, tr, _ = ref.phantom(256, 8, seed=5, height=192).image()
    assert np.array_equal(image, px) and np.array_equal(truth, tr)


@pytest.mark.parametrize("w,h,block,brick", [(256, 256, 8, False), (61, 47, 5, False),
                                             (300, 170, 7, True), (256, 256, 8, True),
                                             (33, 9, 1, False), (40, 40, 3, True)])
def test_oversegment(ctx, w, h, block, brick):
    ctx.make_phantom(w, h, 0.2, 0.0, 0.0, False, 1, copy_out=False)
    R, region = ctx.oversegment(block, brick)
    want, R_host = inputs.oversegment(w, h, block, brick)
    assert R == R_host and np.array_equal(region, want)


def test_errors(ctx):
    with pytest.raises(E.InputError):
        ctx.make_phantom(0, 5)
    with pytest.raises(E.InputError):
        ctx.make_phantom(8, 8, pore_fraction=1.0)
    with pytest.raises(E.InputError):
        ctx.make_phantom(8, 8, sp_rate=1.5)
    with pytest.raises(E.InputError):
        ctx.make_phantom(8, 8, gauss_sigma=-1.0)
    ctx.make_phantom(8, 8, copy_out=False)
    with pytest.raises(E.InputError):
        ctx.oversegment(0)


@pytest.mark.parametrize("size,block,brick,M", [(384, 8, False, 2), (384, 8, True, 5),
                                                (2560, 8, False, 2)])
def test_device_pipeline(ctx, size, block, brick, M):
    info = ctx.synthetic_slice(size, block, brick=brick, seed=9)
    g = ctx.get_graph()
    hd = ctx.get_hoods()
    sl = inputs.synthetic_slice(size, block, brick=brick, seed=9)
    assert np.array_equal(g.offsets, sl.graph.offsets) and np.array_equal(g.neighbors, sl.graph.neighbors)
    assert np.array_equal(g.region_mean, sl.graph.region_mean)
    assert info["regions"] == sl.graph.num_vertices
    cfg = E.OptimizerConfig(num_labels=M, em_max_iters=5, rng_seed=9)
    got = ctx.optimize(cfg, trace_level=E.TRACE_EM, multilabel=M != 2)
    ref = E.Context(0)
    try:
        ref.set_graph(sl.graph)
        ref.build_neighborhoods(sl.cliques)
        assert np.array_equal(ref.get_hoods().members, hd.members)
        want = ref.optimize(cfg, trace_level=E.TRACE_EM, multilabel=M != 2)
    finally:
        ref.close()
    assert np.array_equal(got.labels, want.labels)
    assert np.array_equal(got.mu, want.mu) and np.array_equal(got.sigma, want.sigma)
