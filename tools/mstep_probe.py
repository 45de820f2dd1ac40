"""Phase timeline of the M-step folds on the device-resident loop.

    tools/build_variant.sh probe WORKTREE -DDPMRF_PROBE
    DPMRF_CUDA_LIB=build/variants/probe.so python tools/mstep_probe.py [B|D] [reps]

Runs the bench's config (fixed work), then reads the %globaltimer stamps the
probe build writes (mstep.cu PROBE_*) for the LAST EM iteration's sum-pass
(k=0) and sq-pass (k=1) folds: per block entry / after pdl_wait / staged /
chain done, and the ticket block's ticket / trees / end.  Prints times in us
relative to the sum pass's first block entry."""
import ctypes as ct
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1809_05018_b200 import _native  # noqa: E402
from paper_1809_05018_b200 import engine as E  # noqa: E402

CFG = {"B": (2560, 8, 20), "D": (16384, 7, 2), "A": (256, 8, 10)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "B"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    size, block, em = CFG[name]
    ctx = E.Context(0)
    ctx.synthetic_slice(size, block, seed=42)
    cfg = E.OptimizerConfig(em_max_iters=em, rng_seed=42)
    lib = _native.cuda()
    fn = lib.dpmrf_probe_read
    fn.argtypes = [ct.c_void_p, ct.c_void_p]
    out = []
    for _ in range(reps):
        r = ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_NONE)
        blk = np.zeros((2, 256, 8), np.uint64)
        tail = np.zeros((2, 4), np.uint64)
        assert fn(blk.ctypes.data, tail.ctypes.data) == 0
        valid = [(blk[k][:, 0] > 0) for k in range(2)]
        t0 = int(blk[0][valid[0], 0].min())
        rec = {"optimize_ms": r.stats["optimize_ms"], "em_us": r.stats["optimize_ms"] * 1e3 / em}
        for k, nm in ((0, "sum"), (1, "sq")):
            b = blk[k][valid[k]].astype(np.int64) - t0
            done = b[:, 3][blk[k][valid[k], 3] > 0]
            rec[nm] = {
                "blocks": int(valid[k].sum()),
                "entry_min": float(b[:, 0].min()) / 1e3, "entry_max": float(b[:, 0].max()) / 1e3,
                "wait_min": float(b[:, 1].min()) / 1e3, "wait_max": float(b[:, 1].max()) / 1e3,
                "staged_max": float(b[:, 2].max()) / 1e3,
                "chain_min": float(done.min()) / 1e3 if done.size else None,
                "chain_max": float(done.max()) / 1e3 if done.size else None,
                "ticket": (int(tail[k][0]) - t0) / 1e3, "trees": (int(tail[k][1]) - t0) / 1e3,
                "end": (int(tail[k][2]) - t0) / 1e3,
            }
        for k in range(2):  # per-block: staged -> mid -> after bar -> done (us)
            b = blk[k][valid[k]].astype(np.int64)
            ok = (b[:, 3] > 0) & (b[:, 4] > 0) & (b[:, 5] > 0)
            b = b[ok]
            if not len(b):
                continue
            d0 = (b[:, 4] - b[:, 2]) / 1e3  # issue/mu -> first half landed
            d1 = (b[:, 5] - b[:, 4]) / 1e3  # first span
            d3 = (b[:, 3] - b[:, 5]) / 1e3  # second wait + span
            rec[f"k{k}_first_wait_us"] = [float(np.percentile(d0, q)) for q in (0, 50, 100)]
            rec[f"k{k}_first_span_us"] = [float(np.percentile(d1, q)) for q in (0, 50, 100)]
            rec[f"k{k}_second_us"] = [float(np.percentile(d3, q)) for q in (0, 50, 100)]
            idx = np.nonzero(valid[k])[0][ok]
            slow = idx[(d0 > 1.0) | (d3 > 3.5)]
            rec[f"k{k}_slow_blocks"] = slow.tolist()[:40]
            rec[f"k{k}_per_block"] = [(int(i), round(float(x), 2), round(float(y), 2),
                                       int(blk[k][i][6]), int(blk[k][i][7]))
                                      for i, x, y in zip(idx, d0, d3)]
            rec[f"k{k}_first_wait_hist"] = np.histogram(d0, bins=[0, .5, 1, 1.5, 2, 2.5, 3, 5])[0].tolist()
        b0 = blk[0][valid[0]]
        cyc, ns = b0[:, 6].astype(np.float64), b0[:, 7].astype(np.float64)
        okc = ns > 0
        rec["sum_first_span_cycles_ns_mhz"] = [float(np.median(cyc[okc])), float(np.median(ns[okc])),
                                               float(np.median(cyc[okc] / ns[okc] * 1e3))]
        rec["tail_mu_loads_us"] = (int(tail[0][2]) - t0) / 1e3
        rec["tail_chunks_us"] = (int(tail[0][0]) - t0) / 1e3
        out.append(rec)
        print(json.dumps(rec))
    ctx.close()


if __name__ == "__main__":
    main()
