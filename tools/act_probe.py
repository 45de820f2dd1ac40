"""Items the active-set passes re-evaluate per MAP iteration (probe build):
    DPMRF_CUDA_LIB=build/variants/probe.so python tools/act_probe.py [B|C|D]
prints, per EM iteration of a fixed-work run, the vertices (sparse passes,
t >= 2) and series (t > L) that were flagged."""
import ctypes as ct
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1809_05018_b200 import _native  # noqa: E402
from paper_1809_05018_b200 import engine as E  # noqa: E402

CFG = {"B": (2560, 8, False, 2), "C": (2560, 8, True, 5), "D": (16384, 7, False, 2)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "B"
    size, block, brick, M = CFG[name]
    ctx = E.Context(0)
    ctx.synthetic_slice(size, block, brick=brick, seed=42)
    fn = _native.cuda().dpmrf_probe_read_act
    fn.argtypes = [ct.c_void_p]
    buf = np.zeros((2, 64), np.uint64)
    out = {"config": name, "R": ctx.R}
    for em in (1, 2, 3, 6):
        cfg = E.OptimizerConfig(num_labels=M, em_max_iters=em, rng_seed=42)
        fn(buf.ctypes.data)  # zero
        # only the LAST EM's counts are of interest: run em-1 EMs, zero, run em
        r = ctx.optimize(cfg, fixed_work=True, multilabel=M != 2, trace_level=E.TRACE_NONE,
                         active_set=True)
        fn(buf.ctypes.data)
        out[f"em{em}_total_vertices_per_t"] = buf[0][:10].tolist()
        out[f"em{em}_total_series_per_t"] = buf[1][:10].tolist()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
