"""Structure-phase timing: image + label map -> region graph -> maximal cliques
-> neighborhoods, on the device (csrc/structure.cu, hoods.cu) vs the reference
(oracle/_ref: build_region_graph / enumerate_maximal_cliques / build_neighborhoods
with Backend::threaded(nproc), times measured inside the reference driver).

    python tools/bench_structure.py [--configs B,C,D] [--ref-configs B,C] [--reps 5]

Prints one JSON line per config.  Device times are host wall clock around each
synchronous C-ABI call (the image + label map are copied to the device from
pinned memory first, timed separately), median of --reps after one warm-up."""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1809_05018_b200 import engine as E  # noqa: E402
from paper_1809_05018_b200 import inputs  # noqa: E402

CFG = {"B": (2560, 8, False), "C": (2560, 8, True), "D": (16384, 7, False)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="B,C,D")
    ap.add_argument("--ref-configs", default="B,C")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    ctx = E.Context(0)
    for name in args.configs.split(","):
        size, block, brick = CFG[name]
        spec = inputs.PhantomSpec(size, size, 0.25, 0.05, 100.0, True, 42)
        _, clean = inputs.gen_phantom(spec)
        img = inputs.corrupt(clean, spec)
        reg, R = inputs.oversegment(size, size, block, brick)
        t_host = time.perf_counter()
        g_host = inputs.region_graph(size, size, img, reg, R)
        t_host_graph = time.perf_counter() - t_host
        t_host = time.perf_counter()
        cl_host = inputs.maximal_cliques(g_host)
        t_host_cliques = time.perf_counter() - t_host
        steps = {"h2d_pinned": [], "graph": [], "cliques": [], "hoods": []}
        import torch
        img_pin = torch.from_numpy(img).pin_memory()
        reg_pin = torch.from_numpy(reg.view(np.int32)).pin_memory()
        img_d = torch.empty_like(img_pin, device="cuda")
        reg_d = torch.empty_like(reg_pin, device="cuda")
        for rep in range(args.reps + 1):
            torch.cuda.synchronize()
            t = time.perf_counter()
            img_d.copy_(img_pin, non_blocking=True)
            reg_d.copy_(reg_pin, non_blocking=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            A = ctx.build_region_graph_device(size, size, img_d.data_ptr(), reg_d.data_ptr(), R)
            t1 = time.perf_counter()
            C, CS = ctx.enumerate_maximal_cliques()
            t2 = time.perf_counter()
            S = ctx.build_neighborhoods_resident()
            t3 = time.perf_counter()
            if rep:
                steps["h2d_pinned"].append((t0 - t) * 1e3)
                steps["graph"].append((t1 - t0) * 1e3)
                steps["cliques"].append((t2 - t1) * 1e3)
                steps["hoods"].append((t3 - t2) * 1e3)
        # the whole synthetic slice on the device: phantom + corrupt, oversegmentation
        syn = {"phantom": [], "oversegment": [], "graph": [], "cliques": [], "hoods": []}
        ties = 0
        for rep in range(args.reps + 1):
            t0 = time.perf_counter()
            _, _, ties = ctx.make_phantom(size, size, 0.25, 0.05, 100.0, True, 42, copy_out=False)
            t1 = time.perf_counter()
            ctx.oversegment(block, brick, copy_out=False)
            t2 = time.perf_counter()
            ctx.build_region_graph_resident()
            t3 = time.perf_counter()
            ctx.enumerate_maximal_cliques()
            t4 = time.perf_counter()
            ctx.build_neighborhoods_resident()
            t5 = time.perf_counter()
            if rep:
                for k, a, b in (("phantom", t0, t1), ("oversegment", t1, t2), ("graph", t2, t3),
                                ("cliques", t3, t4), ("hoods", t4, t5)):
                    syn[k].append((b - a) * 1e3)
        # validate_label_map of the (host) label map on the device, H2D included
        val = []
        for rep in range(args.reps + 1):
            t0 = time.perf_counter()
            nreg = ctx.validate_label_map(size, size, reg)
            if rep:
                val.append((time.perf_counter() - t0) * 1e3)
        assert nreg == R
        g = ctx.get_graph()
        cl = ctx.get_cliques()
        same = bool(np.array_equal(g.offsets, g_host.offsets) and
                    np.array_equal(g.neighbors, g_host.neighbors) and
                    np.array_equal(g.region_mean, g_host.region_mean) and
                    np.array_equal(cl.offsets, cl_host.offsets) and
                    np.array_equal(cl.members, cl_host.members))
        line = {"config": name, "size": size, "block": block, "brick": brick, "regions": R,
                "adjacency": A, "cliques": C, "slots": S, "pixels": size * size,
                "device_ms": {k: statistics.median(v) for k, v in steps.items()},
                "host_cpp_builder_s": {"graph": t_host_graph, "cliques": t_host_cliques},
                "device_equals_host_builder": same,
                "h2d_bytes": 5 * size * size,
                "device_synthetic_ms": {k: statistics.median(v) for k, v in syn.items()},
                "device_synthetic_host_ties": ties,
                "device_validate_label_map_ms": statistics.median(val)}
        if name in args.ref_configs.split(","):
            import oracle
            if oracle.ref_available():
                ref = oracle.Ref()
                thr = ref.hw_threads()
                for threads in sorted({1, thr}):
                    p = ref.labelmap(size, size, img, reg, R, threads=threads)
                    t = p.times()
                    line[f"reference_s_threads{threads}"] = {"graph": t[0], "cliques": t[1],
                                                             "hoods": t[2]}
                    del p
                t0 = time.perf_counter()
                assert ref.validate_label_map(size, size, reg) == R
                line["reference_validate_label_map_s"] = time.perf_counter() - t0
        print(json.dumps(line), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
