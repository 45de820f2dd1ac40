"""Regenerate tests/golden/*.npz from the reference itself (oracle/_ref).

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_fixtures.py

Each fixture stores the INPUT (region graph CSR + means, cliques, hoods, all
produced by the reference's own builders) and the reference's OUTPUT of
dpmrf::optimize / the public-step fixed-work recomposition, so the CPU suite
can pin the C restatement and the GPU suite can pin the CUDA path without
/root/reference at run time.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Config, Ref  # noqa: E402

# (name, phantom kwargs, config kwargs, mode, fixed_work)
CASES = [
    # config A of BASELINE.json: 256^2, grid block 8, 2 labels, 10 EM (reference semantics)
    ("configA_256_grid8", dict(size=256, block=8, seed=42),
     dict(rng_seed=42, em_max_iters=10), 0, False),
    # acceptance.cpp:383-426 pipeline: 128^2, block 4, seed 42 (reference semantics)
    ("accept_128_grid4", dict(size=128, block=4, seed=42), dict(rng_seed=42), 0, False),
    # fixed work (no early exits), 3 EM x 10 MAP
    ("fixed_128_grid8", dict(size=128, block=8, seed=7), dict(rng_seed=7, em_max_iters=3), 1, True),
    # 5-label extension on the brick layout (config C shape, small), fixed work
    ("m5_128_brick8", dict(size=128, block=8, seed=42, brick=True),
     dict(num_labels=5, rng_seed=42, em_max_iters=3), 1, True),
    # block 7: region means not dyadic, so fold order matters
    ("configA_252_grid7", dict(size=252, block=7, seed=3), dict(rng_seed=3, em_max_iters=8), 0,
     False),
]


def main():
    ref = Ref()
    for name, pk, ck, mode, fixed in CASES:
        p = ref.phantom(**pk)
        g, h = p.graph(), p.hoods()
        c_off, c_mem = p.cliques()
        cfg = Config(**ck)
        r = p.optimize(cfg, mode=mode, fixed_work=fixed, full_trace=True)
        last = r.trace[-1].map_iters[-1]
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"),
            g_off=g.offsets, g_nbr=g.neighbors, g_mean=g.region_mean, c_off=c_off, c_mem=c_mem,
            h_off=h.offsets, h_mem=h.members,
            cfg=np.array([cfg.num_labels, cfg.em_max_iters, cfg.map_max_iters,
                          cfg.convergence_window], np.int64),
            cfg_f=np.array([cfg.convergence_tol, cfg.beta]), seed=np.uint64(cfg.rng_seed),
            fixed=np.int64(fixed), labels=r.labels, mu=r.mu, sigma=r.sigma,
            em_total=np.array([e.total_energy for e in r.trace]),
            em_conv=np.array([e.converged for e in r.trace], np.uint8),
            em_map_iters=np.array([e.num_map_iters for e in r.trace], np.int64),
            em_mu=np.array([e.mu for e in r.trace]), em_sigma=np.array([e.sigma for e in r.trace]),
            last_hood_energy=last.hood_energy, last_conv=last.converged)
        print(name, "R", p.R, "H", p.H, "S", p.S, "EM", len(r.trace))


if __name__ == "__main__":
    main()
