"""Load the committed reference fixtures (tests/golden/*.npz)."""
import glob
import os

import numpy as np

from oracle import Config, Graph, Hoods

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


class Fixture:
    def __init__(self, name):
        z = np.load(os.path.join(GOLDEN, name + ".npz"))
        self.name = name
        self.z = z
        self.graph = Graph(z["g_off"], z["g_nbr"], z["g_mean"])
        self.hoods = Hoods(z["h_off"], z["h_mem"])
        self.cliques = (z["c_off"], z["c_mem"])
        M, em, mp, L = (int(x) for x in z["cfg"])
        tol, beta = (float(x) for x in z["cfg_f"])
        self.cfg = Config(M, em, mp, L, tol, beta, int(z["seed"]))
        self.fixed = bool(int(z["fixed"]))
        self.multilabel = M != 2

    def check(self, res, exact_trace=True):
        """Assert a Result-like object (labels, mu, sigma, trace) equals the fixture."""
        z = self.z
        assert np.array_equal(np.asarray(res.labels, np.uint32), z["labels"]), self.name
        assert np.array_equal(res.mu, z["mu"]) and np.array_equal(res.sigma, z["sigma"]), self.name
        assert len(res.trace) == len(z["em_total"]), self.name
        for i, e in enumerate(res.trace):
            assert e.total_energy == z["em_total"][i], (self.name, i)
            assert bool(e.converged) == bool(z["em_conv"][i]), (self.name, i)
            assert e.num_map_iters == z["em_map_iters"][i], (self.name, i)
            assert np.array_equal(e.mu, z["em_mu"][i]) and np.array_equal(e.sigma, z["em_sigma"][i])
        if exact_trace and res.trace and res.trace[-1].map_iters:
            last = res.trace[-1].map_iters[-1]
            assert np.array_equal(last.hood_energy, z["last_hood_energy"]), self.name
            assert np.array_equal(last.converged, z["last_conv"]), self.name
