import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from golden_io import Fixture
from paper_1809_05018_b200 import engine as E
f = Fixture(sys.argv[1] if len(sys.argv) > 1 else "m5_128_brick8")
ctx = E.Context(0)
ctx.set_graph(E.RegionGraph(f.graph.offsets, f.graph.neighbors, f.graph.region_mean))
ctx.set_hoods(E.NeighborhoodSet(f.hoods.offsets, f.hoods.members))
c = f.cfg
cfg = E.OptimizerConfig(c.num_labels, c.em_max_iters, c.map_max_iters, c.convergence_window, c.convergence_tol, c.beta, c.rng_seed)
z = f.z
for kw in [dict(), dict(host_log=True), dict(graphs=False), dict(host_log=True, graphs=False), dict(persistent=True, host_log=True)]:
    r = ctx.optimize(cfg, fixed_work=f.fixed, trace_level=E.TRACE_EM, **kw)
    ok = np.array_equal(r.labels, z["labels"])
    print(kw, "labels ok" if ok else f"labels differ at {np.nonzero(r.labels != z['labels'])[0][:10]}",
          "mu", r.mu, "want", z["mu"], "dev_loop", r.stats["device_loop"])
    for i, e in enumerate(r.trace):
        print("   em", i, e.total_energy == z["em_total"][i], e.num_map_iters, np.array_equal(e.mu, z["em_mu"][i]), e.mu - z["em_mu"][i])
