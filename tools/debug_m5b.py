import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from golden_io import Fixture
from oracle import C
from paper_1809_05018_b200 import engine as E
ctx = E.Context(0)
rng = np.random.default_rng(1)
for R in (264, 1000, 20000):
    g_mean = rng.uniform(0, 255, R)
    off = np.zeros(R + 1, np.uint32)
    ctx.set_graph(E.RegionGraph(off, np.zeros(0, np.uint32), g_mean))
    for M in (2, 3, 5):
        labels = rng.integers(0, M, R).astype(np.uint32)
        p = ctx.update_parameters(labels, E.LabelParams(np.zeros(M), np.ones(M)))
        om, os_ = C().update_parameters(g_mean, labels, np.zeros(M), np.ones(M))
        print(R, M, "mu ok" if np.array_equal(p.mu, om) else f"mu BAD {p.mu} vs {om}", "sig ok" if np.array_equal(p.sigma, os_) else "sig BAD")
