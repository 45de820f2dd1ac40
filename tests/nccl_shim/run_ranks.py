"""TEST INFRASTRUCTURE: the NCCL schedule of the partitioned optimize at
world > 1 on ONE GPU.  Every rank is a host thread with its own context
(own stream); csrc/partition.cu binds the in-process shim
(tests/nccl_shim/nccl_shim.cu) through DPMRF_NCCL_LIB instead of libnccl.so.2,
so its grouped halo send/recv, counter all-reduce and in-place all-gathers
run exactly as on N GPUs.  Results must equal the one-device optimize bit for
bit.

    DPMRF_NCCL_LIB=/path/libnccl_shim.so python tests/nccl_shim/run_ranks.py \
        SIZE BLOCK BRICK M WORLD FIXED SEED [SPLIT]
prints one JSON line {"ok": true, ...} or raises."""
import json
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1809_05018_b200 import engine as E  # noqa: E402
from paper_1809_05018_b200 import inputs  # noqa: E402


def main():
    size, block, brick, M, world, fixed, seed = (int(a) for a in sys.argv[1:8])
    assert os.environ.get("DPMRF_NCCL_LIB"), "DPMRF_NCCL_LIB must name the shim"
    sl = inputs.synthetic_slice(size, block, brick=bool(brick), seed=seed)
    cfg = E.OptimizerConfig(num_labels=M, em_max_iters=6, rng_seed=seed)
    ml = M != 2
    base = E.Context(0)
    base.set_graph(sl.graph)
    base.build_neighborhoods(sl.cliques)
    hoods = base.get_hoods()
    want = base.optimize(cfg, fixed_work=bool(fixed), multilabel=ml, trace_level=E.TRACE_EM)
    uid = E.nccl_unique_id()
    assert uid[:4] == b"SHIM", "partition.cu did not bind the shim"
    out, errors = [None] * world, []

    def rank_main(r):
        try:
            ctx = E.Context(0)
            ctx.set_graph(sl.graph)
            ctx.set_hoods(hoods)
            g = E.PartitionGroup.nccl(ctx, uid, r, world)
            res = []
            for _ in range(2):  # twice: state left by one run must not leak into the next
                res.append(g.optimize(cfg, fixed_work=bool(fixed), multilabel=ml))
            out[r] = (res, g.info())
            g.close()
            ctx.close()
        except Exception as ex:  # surfaced below
            errors.append((r, repr(ex)))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise SystemExit(f"rank errors: {errors}")
    for r in range(world):
        for got in out[r][0]:
            assert np.array_equal(got.labels, want.labels), f"rank {r}: labels differ"
            assert np.array_equal(got.params.mu, want.params.mu), f"rank {r}: mu differs"
            assert np.array_equal(got.params.sigma, want.params.sigma), f"rank {r}: sigma differs"
            assert [e.total_energy for e in got.trace] == [e.total_energy for e in want.trace]
            assert [e.num_map_iters for e in got.trace] == [e.num_map_iters for e in want.trace]
    info = out[0][1]
    print(json.dumps({"ok": True, "world": world, "regions": int(base.R), "M": M,
                      "fixed": fixed, "em_iters": len(want.trace),
                      "map_iters": [e.num_map_iters for e in want.trace],
                      "group_info_rank0": {k: (int(v) if isinstance(v, int) else v)
                                           for k, v in info.items()}}))
    base.close()


if __name__ == "__main__":
    main()
