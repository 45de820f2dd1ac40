import sys, ctypes as ct
sys.path.insert(0, ".")
import numpy as np
from paper_1809_05018_b200 import engine as E, _native as N
c = E.Context(0)
c.synthetic_slice(2560, 8, seed=42)
cfg = E.OptimizerConfig(em_max_iters=1, rng_seed=42)
for i in range(3):
    r = c.optimize(cfg, fixed_work=True, trace_level=E.TRACE_NONE)
lib = N.cuda()
buf = (ct.c_ulonglong * 64)()
lib.dpmrf_debug_leaf_prof(buf)
p = list(buf)
for k in (0, 1):
    b = k * 8
    t0 = p[b]
    print("pass", k, "wait %.2f stage %.2f chain %.2f | last-block start %.2f tree %.2f tail %.2f us" % (
        (p[b+1]-t0)/1e3, (p[b+2]-p[b+1])/1e3, (p[b+3]-p[b+2])/1e3, (p[b+4]-t0)/1e3, (p[b+5]-p[b+4])/1e3, (p[b+6]-p[b+5])/1e3))
print("gap pass0 end -> pass1 start %.2f us" % ((p[8] - p[6]) / 1e3))
