"""Phase stamps of k_mstep_stream (probe build, -DDPMRF_PROBE):
    DPMRF_CUDA_LIB=build/variants/probe.so python tools/stream_probe.py [D] [reps]
per block (first 256): entry, after the grid dependency, sum pass done, past
the grid barrier, sq pass done; last block: ticket, end.  Times in us from
the earliest block entry of the last EM iteration."""
import ctypes as ct
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1809_05018_b200 import _native  # noqa: E402
from paper_1809_05018_b200 import engine as E  # noqa: E402

CFG = {"D": (16384, 7, 2), "B4": (4096, 8, 3)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "D"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    size, block, em = CFG[name]
    ctx = E.Context(0)
    ctx.synthetic_slice(size, block, seed=42)
    cfg = E.OptimizerConfig(em_max_iters=em, rng_seed=42)
    fn = _native.cuda().dpmrf_probe_read
    fn.argtypes = [ct.c_void_p, ct.c_void_p]
    for _ in range(reps):
        r = ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_NONE)
        blk = np.zeros((2, 256, 8), np.uint64)
        tail = np.zeros((2, 4), np.uint64)
        assert fn(blk.ctypes.data, tail.ctypes.data) == 0
        b = blk[0][:, :5].astype(np.int64)
        ok = b[:, 0] > 0
        b = b[ok]
        t0 = b[:, 0].min()
        q = lambda c: [round(float(np.percentile((b[:, c] - t0) / 1e3, p)), 2) for p in (0, 50, 100)]  # noqa: E731
        print(json.dumps({"em_us": r.stats["optimize_ms"] * 1e3 / em, "blocks": int(ok.sum()),
                          "entry": q(0), "wait": q(1), "sum_done": q(2), "barrier": q(3),
                          "sq_done": q(4), "tail_ticket": (int(tail[0][0]) - t0) / 1e3,
                          "tail_end": (int(tail[0][1]) - t0) / 1e3}))
    ctx.close()


if __name__ == "__main__":
    main()
