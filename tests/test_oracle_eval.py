"""Evaluation: the oracle's confusion / labels-to-mask
restatement pinned to the reference's own eval tests and to the reference
library (oracle/_ref), and the host-side compute_metrics / porosity of the
Python mirror against the reference's."""
import numpy as np
import pytest

from oracle import Config, OracleError

from paper_1809_05018_b200 import engine as E


def test_confusion_four_quadrants(orc):  # eval_test.cpp:149-169
    truth = [1, 1, 0, 0]
    assert orc.confusion([1, 0, 0, 1], truth) == (1, 1, 1, 1)  # tp tn fp fn
    assert orc.confusion(truth, truth) == (2, 2, 0, 0)
    assert orc.confusion([0, 0, 1, 1], truth) == (0, 0, 2, 2)
    assert orc.confusion([], []) == (0, 0, 0, 0)
    assert orc.confusion([7, 255, 0], [3, 0, 0]) == (1, 1, 1, 0)  # nonzero = positive


def test_confusion_vs_reference(orc, ref):
    rng = np.random.default_rng(3)
    for n in (1, 4, 31, 1000, 65537):
        p = rng.integers(0, 3, n).astype(np.uint8)
        t = rng.integers(0, 2, n).astype(np.uint8)
        assert orc.confusion(p, t) == ref.confusion(n, 1, p, n, 1, t)
    with pytest.raises(OracleError):  # eval_test.cpp:171-176: shapes differ
        ref.confusion(4, 1, np.ones(4, np.uint8), 2, 2, np.ones(4, np.uint8))
    with pytest.raises(E.InputError):  # the mirror raises before any device work
        E.confusion(E.Backend.cuda(), E.BinaryImage(4, 1, np.ones(4, np.uint8)),
                    E.BinaryImage(2, 2, np.ones(4, np.uint8)))


@pytest.mark.parametrize("counts", [(1, 1, 1, 1), (5, 5, 0, 0), (0, 3, 0, 0), (0, 0, 0, 0),
                                    (0, 2, 3, 0), (0, 2, 0, 4), (17, 1000, 3, 9),
                                    (2**40, 3, 2**33, 7)])
def test_compute_metrics_vs_reference(ref, counts):  # eval_test.cpp:178-210
    m = E.compute_metrics(E.ConfusionCounts(*counts))
    want = ref.compute_metrics(counts)
    assert (m.precision, m.recall, m.accuracy, m.precision_defined, m.recall_defined) == want


def test_porosity_vs_reference(ref):
    rng = np.random.default_rng(5)
    for w, h in ((0, 0), (1, 1), (17, 9), (128, 128)):
        px = (rng.random(w * h) < 0.3).astype(np.uint8)
        assert E.porosity(E.BinaryImage(w, h, px)) == ref.porosity(w, h, px)


def test_acceptance_pipeline_quality(orc, ref):
    """acceptance.cpp:383-426 through the reference library: 128^2 phantom,
    block 4, optimize (seed 42), the oracle's labels_to_mask, the reference's
    confusion -> P / R / A >= 0.95 (measured 0.9576 / 0.9735 / 0.9825)."""
    p = ref.phantom(size=128, block=4, seed=42)
    res = p.optimize(Config(rng_seed=42), full_trace=False)
    px, truth, region = p.image()
    mask = orc.labels_to_mask(region, res.labels, res.mu)
    c = ref.confusion(128, 128, mask, 128, 128, truth)
    assert c == orc.confusion(mask, truth)
    m = E.compute_metrics(E.ConfusionCounts(*c))
    assert m.precision >= 0.95 and m.recall >= 0.95 and m.accuracy >= 0.95
    assert round(m.precision, 4) == 0.9576 and round(m.recall, 4) == 0.9735
    assert round(m.accuracy, 4) == 0.9825
