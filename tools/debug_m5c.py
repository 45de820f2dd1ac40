import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from golden_io import Fixture
from oracle import C, Config
from paper_1809_05018_b200 import engine as E
f = Fixture("m5_128_brick8")
ctx = E.Context(0)
ctx.set_graph(E.RegionGraph(f.graph.offsets, f.graph.neighbors, f.graph.region_mean))
ctx.set_hoods(E.NeighborhoodSet(f.hoods.offsets, f.hoods.members))
c = f.cfg
for mm in (1, 2, 3, 10):
    cfg = E.OptimizerConfig(5, 1, mm, min(3, mm - 1) if mm > 1 else 1, c.convergence_tol, c.beta, c.rng_seed)
    if mm == 1:
        cfg.convergence_window = 1; cfg.map_max_iters = 2
    r = ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_EM, host_log=True)
    o = C().optimize(f.graph, f.hoods, Config(5, 1, cfg.map_max_iters, cfg.convergence_window, c.convergence_tol, c.beta, c.rng_seed), fixed_work=True, allow_multilabel=True)
    mu0, sg0, lab0 = C().init_random(5, f.graph.num_vertices, c.rng_seed, True)
    um, us = C().update_parameters(f.graph.region_mean, r.labels, mu0, sg0)
    p = ctx.update_parameters(r.labels, E.LabelParams(mu0, sg0))
    print("map", cfg.map_max_iters, "labels==oracle", np.array_equal(r.labels, o.labels), "mu==oracle", np.array_equal(r.mu, o.mu),
          "mu==orc.update(labels)", np.array_equal(r.mu, um), "dev.update==orc.update", np.array_equal(p.mu, um))
    print("   counts", np.bincount(r.labels, minlength=5), "oracle", np.bincount(o.labels, minlength=5))
    print("   r.mu", r.mu, "\n   um  ", um)
