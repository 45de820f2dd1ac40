import sys, time, statistics
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1809_05018_b200 import engine as E, inputs
size = int(sys.argv[1]) if len(sys.argv) > 1 else 2560
sl = inputs.synthetic_slice(size, 8, seed=42)
ctx = E.Context(0)
ctx.set_graph(sl.graph); ctx.build_neighborhoods(sl.cliques); hd = ctx.get_hoods()
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
g = E.RegionGraph(pin(sl.graph.offsets), pin(sl.graph.neighbors), pin(sl.graph.region_mean))
h = E.NeighborhoodSet(pin(hd.offsets), pin(hd.members))
lab = torch.zeros(len(g.offsets) - 1, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
cfg = E.OptimizerConfig(em_max_iters=20, rng_seed=42)
def a():
    ctx.set_graph(g); ctx.set_hoods(h)
    return ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_NONE, labels_out=lab)
def b():
    return ctx.optimize_arrays(g, h, cfg, fixed_work=True, trace_level=E.TRACE_NONE, labels_out=lab)
def c():
    return ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_NONE, labels_out=lab)
def d():
    ctx.set_graph(g); ctx.set_hoods(h)
cfg0 = E.OptimizerConfig(em_max_iters=0, rng_seed=42)
def e():  # upload + prepare + no EM
    return ctx.optimize_arrays(g, h, cfg0, fixed_work=True, trace_level=E.TRACE_NONE, labels_out=lab)
res = {"sethoods+optimize": [], "optimize_arrays": [], "optimize_only": [], "upload_only": [],
       "arrays_em0": []}
for f in (a, b, c, d, e): f(); f()
for rep in range(30):
    for name, f in (("sethoods+optimize", a), ("optimize_arrays", b), ("optimize_only", c),
                    ("upload_only", d), ("arrays_em0", e)):
        torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); res[name].append((time.perf_counter() - t0) * 1e3)
        if name == "optimize_only": dev = r.stats["optimize_ms"]
for k, v in res.items(): print(k, "median %.3f ms  min %.3f" % (statistics.median(v), min(v)))
print("device optimize_ms", dev)
