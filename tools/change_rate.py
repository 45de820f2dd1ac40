"""Labels changed per MAP iteration (EM iterations 1 and 5) on the benched
slices: how sparse the MAP updates become (design probe for active sets).
    python tools/change_rate.py [B|D]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1809_05018_b200 import engine as E  # noqa: E402

CFG = {"B": (2560, 8), "D": (16384, 7)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "B"
    size, block = CFG[name]
    ctx = E.Context(0)
    ctx.synthetic_slice(size, block, seed=42)
    R = ctx.R
    out = {"config": name, "R": R}
    for em in (1, 5):
        prev = None
        rates = []
        for m in range(2, 12):
            cfg = E.OptimizerConfig(em_max_iters=em, map_max_iters=m, rng_seed=42, convergence_window=1)
            r = ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_NONE)
            lab = np.asarray(r.labels).copy()
            if prev is not None:
                rates.append(int((lab != prev).sum()))
            prev = lab
        out[f"em{em}_changed_per_map_iter"] = rates
    print(json.dumps(out))
    ctx.close()


if __name__ == "__main__":
    main()
