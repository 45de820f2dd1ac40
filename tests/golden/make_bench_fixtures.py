"""Compact fixtures for the EXACT benched workloads (BASELINE.json configs B, C, D),
produced by the reference itself (oracle/_ref, compiled from /root/reference).

    make -C oracle && python tests/golden/make_bench_fixtures.py [B C D ...]

The inputs are too large to commit, so a fixture stores digests instead:

* input: SHA-256 of the reference-built region graph (offsets, neighbors,
  region_mean bytes) and neighborhoods (offsets, members) -- the GPU test
  rebuilds the slice with the device synth + structure builders and must hit
  the same digests before it optimizes;
* output of the public-step fixed-work recomposition of dpmrf::optimize
  (optimize.cpp:31-74 without the two breaks; ref_driver.cpp optimize_steps,
  Backend::threaded): SHA-256 of the labels (u32), per-label counts, exact
  mu / sigma bits, and per EM iteration the total energy, mu, sigma, flags and
  a SHA-256 over every MAP iteration's hood-energy row + convergence flags.

Cases (bench.py CONFIGS): B = 2560^2 grid block 8, M=2, fixed 20 EM x 10 MAP
(the headline step exactly as timed); C = 2560^2 brick block 8, M=5, fixed
3 EM; D = 16384^2 grid block 7, M=2, fixed 2 EM.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Config, Ref  # noqa: E402

CASES = {
    "B": dict(size=2560, block=8, brick=False, seed=42, M=2, em=20),
    "C": dict(size=2560, block=8, brick=True, seed=42, M=5, em=3),
    "D": dict(size=16384, block=7, brick=False, seed=42, M=2, em=2),
}
OUT = os.path.join(HERE, "bench_shapes.json")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def bits(x):
    return [f"{int(v):016x}" for v in np.asarray(x, np.float64).view(np.uint64)]


def trace_digest(em_log):
    """SHA-256 over one EM iteration's MAP rows (hood energy bits, then flags)."""
    h = hashlib.sha256()
    for m in em_log.map_iters:
        h.update(np.ascontiguousarray(m.hood_energy, np.float64).tobytes())
        h.update(np.ascontiguousarray(m.converged, np.uint8).tobytes())
    return h.hexdigest()


def make(name, threads):
    c = CASES[name]
    ref = Ref()
    t0 = time.time()
    p = ref.phantom(c["size"], c["block"], brick=c["brick"], seed=c["seed"], threads=threads)
    g, h = p.graph(), p.hoods()
    t_build = time.time() - t0
    cfg = Config(num_labels=c["M"], rng_seed=c["seed"], em_max_iters=c["em"])
    t0 = time.time()
    r = p.optimize(cfg, threads=threads, mode=1, fixed_work=True, full_trace=True)
    t_opt = time.time() - t0
    assert len(r.trace) == c["em"]
    rec = {
        "case": c, "map_max_iters": cfg.map_max_iters, "convergence_window": cfg.convergence_window,
        "R": p.R, "A": p.A, "H": p.H, "S": p.S,
        "input": {"g_off": sha(g.offsets), "g_nbr": sha(g.neighbors), "g_mean": sha(g.region_mean),
                  "h_off": sha(h.offsets), "h_mem": sha(h.members)},
        "labels_sha256": sha(np.asarray(r.labels, np.uint32)),
        "label_counts": np.bincount(r.labels, minlength=c["M"]).tolist(),
        "mu": bits(r.mu), "sigma": bits(r.sigma),
        "em": [{"total_energy": bits([e.total_energy])[0], "converged": bool(e.converged),
                "num_map_iters": int(e.num_map_iters), "mu": bits(e.mu), "sigma": bits(e.sigma),
                "map_rows_sha256": trace_digest(e)} for e in r.trace],
        "generated_by": "oracle/_ref optimize_steps (Backend::threaded(%d)), fixed work" % threads,
        "seconds": {"reference_structure_build": round(t_build, 1),
                    "reference_optimize": round(t_opt, 1)},
    }
    print(name, "R", p.R, "H", p.H, "S", p.S, f"build {t_build:.1f}s optimize {t_opt:.1f}s",
          flush=True)
    return rec


def main():
    names = sys.argv[1:] or sorted(CASES)
    threads = min(8, os.cpu_count() or 1)
    db = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            db = json.load(f)
    for n in names:
        db[n] = make(n, threads)
        with open(OUT, "w") as f:
            json.dump(db, f, indent=1, sort_keys=True)
            f.write("\n")


if __name__ == "__main__":
    main()
