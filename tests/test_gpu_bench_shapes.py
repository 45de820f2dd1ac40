"""The EXACT benched workloads vs the reference itself (tests/golden/bench_shapes.json,
made by tests/golden/make_bench_fixtures.py from oracle/_ref).

Each case rebuilds its slice with the device synth + structure builders (the
digests of the region graph and neighborhoods must equal the reference
build), then runs the bench's own call -- Context.optimize(fixed_work=True,
TRACE_NONE) on the device-resident loop, i.e. the kernel instances bench.py
times: B = k_map_fused one vertex per thread with the merged M-step tail;
C = the 12-slot brick hood rows at M=5; D = two vertices per thread
(R >= 2^20), the many-block label-tile scan and the chunked M-step trees --
and compares labels (SHA-256), mu/sigma (bits), and per EM iteration the total
energy, parameters, flags and a digest of every MAP iteration's hood-energy
row and flags.  D also runs through the 2-partition schedule (local
transport).  Reference: optimize.cpp:31-74 (fixed work = the two breaks
removed), optimize_test.cpp:125-135 (every backend is bit-identical).
"""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

E = pytest.importorskip("paper_1809_05018_b200.engine")

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "bench_shapes.json")) as _f:
    SHAPES = json.load(_f)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def bits(x):
    return [f"{int(v):016x}" for v in np.asarray(x, np.float64).view(np.uint64)]


def trace_digest(em_log):
    h = hashlib.sha256()
    for m in em_log.map_iters:
        h.update(np.ascontiguousarray(m.hood_energy, np.float64).tobytes())
        h.update(np.ascontiguousarray(m.converged, np.uint8).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    c = E.Context(0)
    yield c
    c.close()


def build(ctx, rec):
    c = rec["case"]
    ctx.synthetic_slice(c["size"], c["block"], brick=c["brick"], seed=c["seed"])
    g = ctx.get_graph(sizes=False)
    h = ctx.get_hoods()
    got = {"g_off": sha(g.offsets), "g_nbr": sha(g.neighbors), "g_mean": sha(g.region_mean),
           "h_off": sha(h.offsets), "h_mem": sha(h.members)}
    assert got == rec["input"], "device-built slice differs from the reference build"
    cfg = E.OptimizerConfig(num_labels=c["M"], em_max_iters=c["em"],
                            map_max_iters=rec["map_max_iters"], rng_seed=c["seed"])
    return cfg


def check_result(rec, r, level):
    assert sha(np.asarray(r.labels, np.uint32)) == rec["labels_sha256"]
    assert bits(r.mu) == rec["mu"] and bits(r.sigma) == rec["sigma"]
    if level == E.TRACE_NONE:
        return
    assert len(r.trace) == len(rec["em"])
    for e, want in zip(r.trace, rec["em"]):
        assert bits([e.total_energy])[0] == want["total_energy"]
        assert bool(e.converged) == want["converged"]
        assert e.num_map_iters == want["num_map_iters"]
        assert bits(e.mu) == want["mu"] and bits(e.sigma) == want["sigma"]
        if level == E.TRACE_FULL:
            assert trace_digest(e) == want["map_rows_sha256"]


@pytest.mark.parametrize("name", sorted(SHAPES))
def test_bench_shape_vs_reference(ctx, name):
    rec = SHAPES[name]
    cfg = build(ctx, rec)
    multilabel = rec["case"]["M"] != 2
    # the timed call of bench.py (device-resident loop, no trace)
    r = ctx.optimize(cfg, fixed_work=True, multilabel=multilabel, trace_level=E.TRACE_NONE)
    assert r.stats["device_loop"] == 1
    check_result(rec, r, E.TRACE_NONE)
    assert np.bincount(r.labels, minlength=rec["case"]["M"]).tolist() == rec["label_counts"]
    # EM-level trace on the same loop, then the full per-MAP trace
    for level in (E.TRACE_EM, E.TRACE_FULL):
        r = ctx.optimize(cfg, fixed_work=True, multilabel=multilabel, trace_level=level)
        check_result(rec, r, level)
    # the active-set MAP loop (extension) reproduces the same fixture
    r = ctx.optimize(cfg, fixed_work=True, multilabel=multilabel, trace_level=E.TRACE_EM,
                     active_set=True)
    assert r.stats["active_set"] == (1 if rec["case"]["M"] == 2 else 0)
    check_result(rec, r, E.TRACE_EM)


@pytest.mark.skipif("D" not in SHAPES, reason="no D fixture")
def test_bench_shape_D_partitioned(ctx):
    """Config D through the vertex-range partition schedule (2 parts, local
    transport: the NCCL schedule's halos as device copies) -- same fixture."""
    rec = SHAPES["D"]
    cfg = build(ctx, rec)
    grp = E.PartitionGroup.local(ctx, 2)
    try:
        r = grp.optimize(cfg, fixed_work=True, multilabel=False, trace_level=E.TRACE_EM)
    finally:
        grp.close()
    check_result(rec, r, E.TRACE_EM)
