"""validate_label_map on the device (labelmap.cu) against the oracle: same
num_regions or the same InputError message, on the shared cases and on large
maps; read_rlm round trip with validation (graph_test.cpp:139-157)."""
import numpy as np
import pytest

from labelmap_cases import cases
from paper_1809_05018_b200 import engine as E

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    c = E.Context(0)
    yield c
    c.close()


def _device(ctx, w, h, region):
    try:
        return ctx.validate_label_map(w, h, region)
    except E.InputError as e:
        return str(e).split(": ", 1)[1]  # strip the "validate_label_map: " prefix


@pytest.mark.parametrize("name,w,h,region", cases(), ids=[c[0] for c in cases()])
def test_validate_vs_oracle(ctx, orc, name, w, h, region):
    assert _device(ctx, w, h, region) == orc.validate_label_map(w, h, region)


def test_empty_map(ctx):
    assert _device(ctx, 0, 4, np.zeros(0, np.uint32)) == "label map: empty"


@pytest.mark.parametrize("kind", ["grid", "brick", "snake", "split_late", "hole"])
def test_large_maps(ctx, orc, kind):
    from paper_1809_05018_b200 import inputs
    w, h = 2048, 1536
    if kind in ("grid", "split_late", "hole"):
        reg, _ = inputs.oversegment(w, h, 7, False)
    elif kind == "brick":
        reg, _ = inputs.oversegment(w, h, 8, True)
    else:
        # one long boustrophedon region through the image plus stripes: the
        # union-find sees chains spanning the whole map
        reg = np.zeros((h, w), np.uint32)
        reg[1::4, :-1] = 1
        reg[3::4, 1:] = 1
        reg = reg.reshape(-1)
    if kind == "split_late":
        reg = reg.copy()
        reg[-1] = reg[w * 7 + 3]  # a late pixel joins an early region
    if kind == "hole":
        reg = reg.copy()
        reg[reg == 5] = 4  # id 5 unused
    assert _device(ctx, w, h, reg) == orc.validate_label_map(w, h, reg)


def test_read_rlm_round_trip(tmp_path):  # graph_test.cpp:139-157
    from paper_1809_05018_b200 import inputs
    reg, R = inputs.oversegment(7, 5, 2, False)
    path = str(tmp_path / "m.rlm")
    E.write_rlm(E.LabelMap(7, 5, reg), path)
    back = E.read_rlm(path)
    assert (back.width, back.height, back.num_regions) == (7, 5, R)
    assert np.array_equal(back.region, reg)
    with open(path, "wb") as f:  # ids 0 and 2 with 1 unused
        f.write(b"RLM1\x02\x00\x00\x00\x01\x00\x00\x00\x00\x00\x00\x00\x02\x00\x00\x00")
    with pytest.raises(E.InputError):
        E.read_rlm(path)


def test_rlm_pipeline_to_mask(ctx, orc, tmp_path):
    """A label map from disk through the whole path: read_rlm (validated on
    the device) -> region graph from host arrays -> cliques -> hoods ->
    optimize -> segment write-back over the uploaded map == the oracle's."""
    from paper_1809_05018_b200 import inputs
    truth, image, _ = ctx.make_phantom(300, 200, 0.25, 0.05, 100.0, True, 77)
    reg, R = inputs.oversegment(300, 200, 6, True)
    path = str(tmp_path / "brick.rlm")
    E.write_rlm(E.LabelMap(300, 200, reg), path)
    lm = E.read_rlm(path)
    assert lm.num_regions == R
    ctx.build_region_graph(lm.width, lm.height, image, lm.region, lm.num_regions)
    ctx.enumerate_maximal_cliques()
    ctx.build_neighborhoods_resident()
    res = ctx.optimize(E.OptimizerConfig(rng_seed=77), trace_level=E.TRACE_NONE)
    mask, none = ctx.segment_mask(res.labels, res.mu, counts=False)
    assert none is None
    want = orc.labels_to_mask(reg, res.labels, res.mu)
    assert np.array_equal(mask, want)
    c = ctx.confusion(mask, truth)
    assert (c.tp, c.tn, c.fp, c.fn) == orc.confusion(want, truth)
    with pytest.raises(ValueError):  # no phantom truth behind an uploaded map
        ctx.segment_mask(res.labels, res.mu)
