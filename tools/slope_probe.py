"""Per-MAP-iteration and per-EM fixed costs of optimize() from timing slopes.

Times fixed-work optimize() (device loop, CUDA graphs, no per-kernel events)
on one slice for several map_max_iters and em_max_iters values; the slope
over MAP iterations is the real (overlapped) cost of one MAP launch, the
intercept per EM the M-step + EM bookkeeping.
usage: python tools/slope_probe.py [size] [block]"""
import sys

import numpy as np

from paper_1809_05018_b200 import engine as E
from paper_1809_05018_b200 import inputs

size = int(sys.argv[1]) if len(sys.argv) > 1 else 2560
block = int(sys.argv[2]) if len(sys.argv) > 2 else 8
flags = sys.argv[3:] if len(sys.argv) > 3 else []
sl = inputs.synthetic_slice(size, block, seed=42)
ctx = E.Context(0)
ctx.set_graph(sl.graph)
ctx.build_neighborhoods(sl.cliques)
kw = {"fused": "unfused" not in flags}
res = {}
for em in (10, 20):
    for mp in (4, 6, 8, 10, 12, 16):
        cfg = E.OptimizerConfig(em_max_iters=em, map_max_iters=mp, rng_seed=42)
        ts = []
        for _ in range(7):
            r = ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_NONE, **kw)
            ts.append(r.stats["optimize_ms"])
        res[(em, mp)] = float(np.median(ts[2:]))
for em in (10, 20):
    mps = np.array([4, 6, 8, 10, 12, 16])
    t = np.array([res[(em, m)] for m in mps])
    a, b = np.polyfit(mps, t, 1)
    print(f"size {size} block {block} em {em}: per-MAP-iteration {a / em * 1e3:.2f} us, "
          f"per-EM fixed {b / em * 1e3:.2f} us  "
          + " ".join(f"{m}:{x:.3f}ms" for m, x in zip(mps, t)))
