#!/usr/bin/env python
"""Benchmark of the DPP-PMRF optimization phase on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config A|B|C|D|E] [--impl ours|reference]

A step is one optimization of one synthetic slice whose region graph and
device-built neighborhoods are resident in HBM: fixed work (20 EM x 10 MAP
iterations, no early exits) for configs B-E, the reference's own semantics
(10 EM, early exits) for config A.  The default line is config B (the
headline: 2560^2 on one B200).

N>1: when WORLD_SIZE is unset, ``--gpus N`` re-launches itself as N ranks
(torch.distributed.run, one process per GPU).  Each rank optimizes its own
config-B slice (seed 42 + rank: slices shard with no data-path collective,
"weak"), so the N=1 line is the same measurement as BENCH; the line then
carries two sub-records of the BASELINE.json multi-GPU configs:
  * "stack_E": the 64-slice stack dealt round-robin to the N ranks (total work
    fixed: strong scaling), no collective on the data path;
  * "partitioned_D": the 16384^2 slice partitioned by vertex range across the
    N ranks (NCCL label/minima halos per MAP iteration, per-EM allgathers),
    checked bit-exact against a one-rank run of the same slice.

value  = EM iterations of all ranks / max-over-ranks device time (CUDA events
         on the library's stream, L2 flushed between steps)
e2e    = the same metric through the public C ABI with host (pinned) buffers:
         one dpmrf_optimize_arrays call per step (optimize(graph, hoods,
         config), engine.hpp:99-100), host wall clock, H2D of the graph and
         hoods and D2H of labels/params included.  e2e_full_trace: the same
         call with the reference's full per-MAP trace (OptimizeResult.trace,
         engine.hpp:82-99) streamed into caller-owned pinned buffers.
--impl reference times the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference by oracle/Makefile) on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MRF opt. EM-iterations/s & vertex-label evals/s @1/2/4/8 B200; %HBM peak"
PHANTOM = "porous phantom (pore .25, s&p .05, gauss 100, ringing)"
CONFIGS = {
    "A": dict(size=256, block=8, brick=False, M=2, em=10, fixed=False,
              desc=f"synthetic 256x256 {PHANTOM}, grid oversegmentation block 8, 2 labels, "
                   "10 EM x 10 MAP with the reference's early exits (seed 42)"),
    "B": dict(size=2560, block=8, brick=False, M=2, em=20, fixed=True,
              desc=f"synthetic 2560x2560 {PHANTOM}, grid oversegmentation block 8, 2 labels, "
                   "fixed 20 EM x 10 MAP (seed 42 + rank)"),
    "C": dict(size=2560, block=8, brick=True, M=5, em=20, fixed=True,
              desc="same 2560x2560 slice, brick oversegmentation block 8 (dense 3-clique graph), "
                   "5 labels, fixed 20 EM x 10 MAP (seed 42)"),
    "D": dict(size=16384, block=7, brick=False, M=2, em=20, fixed=True,
              desc=f"single 16384x16384 {PHANTOM}, grid block 7 (~5.5M regions), 2 labels, "
                   "fixed 20 EM x 10 MAP (seed 42)"),
    "E": dict(size=2560, block=8, brick=False, M=2, em=20, fixed=True,
              desc="64-slice stack of 2560x2560 config-B slices (seed 42+z), fixed 20 EM x 10 MAP "
                   "per slice, slices dealt round-robin to ranks"),
}
MAP_ITERS = 10
L_WINDOW = 3


E2E_WARM_S = float(os.environ.get("DPMRF_E2E_WARM_S", "0.5"))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def host_cpu():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def map_bytes(R, A, H, S, L=L_WINDOW):
    """SURVEY.md §8(d) algorithmic bytes of one MAP iteration (reference dtypes):
    vertex part 20R + 4A + 4, hood part 4(H+1) + 4S + 8H + 8LH."""
    return 20 * R + 4 * A + 4, 4 * (H + 1) + 4 * S + 8 * H + 8 * L * H


def run_bytes(R, A, H, S, em, maps=MAP_ITERS):
    """Algorithmic bytes of one fixed-work optimize: em*maps*B_MAP + em*B_EM,
    B_EM = 24R + 8H (two M-step passes over labels + means, total-energy read)."""
    v, h = map_bytes(R, A, H, S)
    return em * maps * (v + h) + em * (24 * R + 8 * H)


# ---- clocks sampled during the timed region ------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.lines = device, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- the reference CPU path (oracle/_ref = the reference compiled from its sources) ----
def _timed(run, seconds_budget, max_samples=50):
    times = []
    t_end = time.perf_counter() + seconds_budget
    while True:
        t0 = time.perf_counter()
        out = run()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end or len(times) >= max_samples:
            return times, out


def reference_sample(cfg_name, seconds_budget=12.0, rank_seed=42):
    """The reference's fastest CPU path on a bounded sample of the workload.
    Returns (EM-iterations/s, detail).  Fixed-work configs: one EM iteration
    (10 MAP, no early exits) per sample; config A: the whole run as-is."""
    c = CONFIGS[cfg_name]
    import oracle
    em = c["em"] if not c["fixed"] else 1
    if oracle.ref_available():
        kind = "reference"
        ref = oracle.Ref()
        threads = ref.hw_threads()
        pipe = ref.phantom(c["size"], c["block"], brick=c["brick"], seed=rank_seed,
                           threads=min(threads, 8))
        cfg1 = oracle.Config(num_labels=c["M"], rng_seed=rank_seed, em_max_iters=em)
        mode = 1 if (c["fixed"] or c["M"] != 2) else 0
        sweep = lambda: pipe.sweep(cfg1, mode=mode, fixed_work=c["fixed"])  # noqa: E731
        dpp = lambda: pipe.optimize(cfg1, threads=threads, mode=mode,  # noqa: E731
                                    fixed_work=c["fixed"], full_trace=False)
        # fastest of: Algorithm-1 sweep on 1 core, and the DPP engine on all cores
        t0 = time.perf_counter()
        r_s = sweep()
        sweep_rate = len(r_s.trace) / (time.perf_counter() - t0)
        t0 = time.perf_counter()
        r_d = dpp()
        dpp_rate = len(r_d.trace) / (time.perf_counter() - t0)
        best = "sweep" if sweep_rate >= dpp_rate else "dpp"
        run = sweep if best == "sweep" else dpp
        cores = 1 if best == "sweep" else threads
        what = ("optimize_reference sweep (1 core)" if best == "sweep"
                else f"optimize DPP engine (threaded x{threads})")
        sample_desc = (f"config {cfg_name}: {em} EM iteration(s) per sample "
                       f"({'fixed work, ' if c['fixed'] else 'early exits, '}10 MAP) of {what}; "
                       f"probe: sweep {sweep_rate:.3f} EM-it/s, DPP x{threads} {dpp_rate:.3f} EM-it/s")
    else:
        kind = "port"
        from oracle import C, Config, Graph
        from paper_1809_05018_b200 import inputs
        sl = inputs.synthetic_slice(c["size"], c["block"], brick=c["brick"], seed=rank_seed)
        g = Graph(sl.graph.offsets, sl.graph.neighbors, sl.graph.region_mean)
        h, _ = C().build_neighborhoods(g, sl.cliques.offsets, sl.cliques.members)
        cfg1 = Config(num_labels=c["M"], rng_seed=rank_seed, em_max_iters=em)
        run = lambda: C().optimize_reference(g, h, cfg1, fixed_work=c["fixed"],  # noqa: E731
                                             allow_multilabel=True)
        cores = 1
        sample_desc = f"config {cfg_name}: {em} EM iteration(s) of the C port of the sweep, 1 core"
    times, out = _timed(run, seconds_budget)
    ems = len(out.trace) if out.trace else em
    per_em = statistics.median(times) / ems
    return 1.0 / per_em, {"kind": kind, "cores": cores,
                          "sample": sample_desc + f"; {len(times)} samples, median",
                          "run": run, "em_per_run": ems, **host_cpu()}


def reference_sample_stack(slices=64, seconds_budget=12.0):
    """Config E on the CPU: independent optimize_reference sweeps (serial by
    design, no shared state) across all host threads, one slice per thread
    (SURVEY.md §8(d)(iii)).  Sample: nproc slices (seed 42+z), 1 EM iteration
    (10 MAP, fixed work) each, run concurrently; the aggregate rate applies to
    the whole 64-slice stack."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    if not oracle.ref_available():
        return None
    ref = oracle.Ref()
    n = max(1, min(ref.hw_threads(), slices))
    c = CONFIGS["E"]
    with ThreadPoolExecutor(n) as pool:  # (ctypes calls release the GIL)
        pipes = list(pool.map(lambda z: ref.phantom(c["size"], c["block"], seed=42 + z, threads=1),
                              range(n)))
        cfgs = [oracle.Config(rng_seed=42 + z, em_max_iters=1) for z in range(n)]

        def step():
            list(pool.map(lambda z: pipes[z].sweep(cfgs[z], mode=1, fixed_work=True), range(n)))
        times, _ = _timed(step, seconds_budget, max_samples=20)
    per = statistics.median(times)
    return n / per, {"kind": "reference", "cores": n,
                     "sample": f"config E: {n} slices (seed 42+z) x 1 EM iteration (10 MAP, fixed "
                               f"work) of optimize_reference, one slice per host thread, run "
                               f"concurrently; {len(times)} samples, median", **host_cpu()}


def reference_sample_arrays(g, h, M, em=1):
    """optimize_reference on the given (device-built, reference-identical) slice:
    one EM iteration, fixed work, 1 core (used for config D, whose reference
    structure build alone takes ~1 min)."""
    import oracle
    if not oracle.ref_available():
        return None
    ref = oracle.Ref()
    pipe = ref.arrays(oracle.Graph(g.offsets, g.neighbors, g.region_mean),
                      hoods=oracle.Hoods(h.offsets, h.members))
    cfg = oracle.Config(num_labels=M, rng_seed=42, em_max_iters=em)
    t0 = time.perf_counter()
    pipe.sweep(cfg, mode=1, fixed_work=True)
    dt = time.perf_counter() - t0
    return em / dt, {"kind": "reference", "cores": 1,
                     "sample": f"config D: {em} EM iteration (10 MAP, fixed work) of "
                               "optimize_reference on the device-built slice (digest-equal to "
                               "the reference build), 1 core, one sample", **host_cpu()}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    _, det = reference_sample(args.config if args.config != "E" else "B", seconds_budget=1.0)
    run = det["run"]
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    per_em = sum(times) / len(times) / det["em_per_run"]
    value = 1.0 / per_em
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "EM-iterations/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sum(times) / len(times) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIGS[args.config]["desc"], "sample": det["sample"]},
            "cpu_baseline": {"value": value, "unit": "EM-iterations/s", "cores": det["cores"],
                             "kind": det["kind"], "sample": det["sample"],
                             "nproc": det["nproc"], "cpu_model": det["cpu_model"]},
            "e2e": {"value": value, "unit": "EM-iterations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---- distributed plumbing ----------------------------------------------------------------
class Dist:
    def __init__(self, torch, dist):
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # DPMRF_BENCH_SHARED_GPU=1 (testing the multi-rank plumbing on a one-GPU
        # box): every rank uses device local % device_count and the gloo backend
        # for the timing collectives (NCCL refuses two ranks on one device).
        self.shared = os.environ.get("DPMRF_BENCH_SHARED_GPU") == "1"
        if self.shared:
            self.local %= torch.cuda.device_count()
        torch.cuda.set_device(self.local)
        if self.world > 1:
            if self.shared:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        self.coll_dev = "cpu" if self.shared else "cuda"

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def _reduce(self, x, op):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.coll_dev)
        self.dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x):
        return self._reduce(x, self.dist.ReduceOp.MAX)

    def sum(self, x):
        return self._reduce(x, self.dist.ReduceOp.SUM)

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def roofline(kname, kbytes, kavg_ms, traffic=None, note=""):
    hbm, peak_kind = peaks()
    achieved = kbytes / (kavg_ms * 1e-3) / 1e9
    return {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": hbm,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
            "algorithmic_bytes_per_launch": kbytes, "avg_launch_us": kavg_ms * 1e3,
            # the same launch time against the ncu-measured DRAM bytes (packed
            # structure + u8 labels move fewer bytes than the reference-dtype
            # algorithmic count, so frac can pass 1)
            "dram_frac": (traffic / (kavg_ms * 1e-3) / 1e9 / hbm) if traffic else None,
            "timing": "profiled pass: CUDA events on the library stream around each EM's chain "
                      "of fused launches (PDL overlap kept), / launches", "note": note}


def ncu_traffic(cfg_name, kname):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(cfg_name, {}).get(kname)
    except Exception:
        return None


# ---- one slice per rank (configs A-D; B is the headline) ---------------------------------
def run_slice(args, E, torch, d: Dist):
    c = CONFIGS[args.config]
    seed = 42 + d.rank if args.config == "B" else 42
    ctx = E.Context(d.local)
    t0 = time.perf_counter()
    info = ctx.synthetic_slice(c["size"], c["block"], brick=c["brick"], seed=seed)
    build_inputs_s = time.perf_counter() - t0
    R, A = info["regions"], info["adjacency"]
    graph_host = ctx.get_graph(sizes=False)  # host copies for the e2e leg
    hoods = ctx.get_hoods()
    H, S = hoods.size(), hoods.total_slots()
    M = c["M"]
    cfg = E.OptimizerConfig(num_labels=M, em_max_iters=c["em"], map_max_iters=MAP_ITERS,
                            rng_seed=seed)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    labels_out = np.zeros(R, np.uint32)
    fixed, ml = c["fixed"], M != 2

    act = getattr(args, "active_set", False)

    def step(timing=False):
        return ctx.optimize(cfg, fixed_work=fixed, multilabel=ml, trace_level=E.TRACE_NONE,
                            kernel_timing=timing, labels_out=labels_out, active_set=act)

    for _ in range(args.warmup):  # the timed configuration (graphs captured here, not timed)
        step()
    sampler = ClockSampler(d.local)
    sampler.start()
    d.barrier()
    dev_ms, launches, ems, maps = [], 0, 0, 0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        r = step()
        dev_ms.append(r.stats["optimize_ms"])
        launches += r.stats["kernel_launches"]
        ems += r.stats["em_iters"]
        maps += r.stats["map_iters_total"]
    d.barrier()
    clocks = sampler.stop()
    # profiled pass (same workload, CUDA events around the MAP loop / M-step
    # of every EM iteration) for the kernel split and the roofline
    prof = {"map_loop_ms": 0.0, "map_loop_launches": 0, "mstep_ms": 0.0, "optimize_ms": 0.0,
            "em_iters": 0}
    prof_steps = max(2, args.steps // 2)
    for _ in range(prof_steps):
        flush.zero_()
        torch.cuda.synchronize()
        st = step(timing=True).stats
        for k in prof:
            prof[k] += st[k]
    total_dev_s = d.max(sum(dev_ms) / 1e3)
    total_em = d.sum(ems)
    value = total_em / total_dev_s
    ms_per_step = total_dev_s * 1e3 / args.steps

    # ---- e2e: public C ABI with host (pinned) buffers --------------------------------
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    g_pin = E.RegionGraph(pin(graph_host.offsets), pin(graph_host.neighbors),
                          pin(graph_host.region_mean))
    h_pin = E.NeighborhoodSet(pin(hoods.offsets), pin(hoods.members))
    lab_pin = torch.zeros(R, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
    h2d = 4 * (R + 1) + 4 * A + 8 * R + 4 * (H + 1) + 4 * S
    d2h = 4 * R + 16 * M

    calls_ms = []  # per-call wall times of each e2e leg (sorted), for the record

    def e2e_leg(trace_level, sink=None, n=max(3, args.steps)):
        call = lambda: ctx.optimize_arrays(g_pin, h_pin, cfg, fixed_work=fixed,  # noqa: E731
                                           multilabel=ml, trace_level=trace_level,
                                           labels_out=lab_pin, trace_sink=sink,
                                           active_set=act)
        # untimed warm-up: W calls and at least E2E_WARM_S of back-to-back calls
        # (the host->device DMA of a fresh process reaches its steady rate
        # only after some traffic: the upload alone measured 0.30-0.36 ms
        # right after a 3-call warm-up vs 0.228 ms later in the same process)
        t_w, k = time.perf_counter(), 0
        while k < args.warmup or time.perf_counter() - t_w < E2E_WARM_S:
            call()
            k += 1
        d.barrier()
        times, devs, em_n = [], [], 0
        for _ in range(n):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            # the reference-facing call: optimize(graph, hoods, config) on host arrays
            r = call()
            times.append(time.perf_counter() - t0)
            em_n += r.stats["em_iters"]
            devs.append(r.stats["optimize_ms"])
        d.barrier()
        up = []  # the H2D of the inputs alone (set_graph + set_hoods, synchronous)
        for _ in range(5):
            t0 = time.perf_counter()
            ctx.set_graph(g_pin)
            ctx.set_hoods(h_pin)
            up.append(time.perf_counter() - t0)
        calls_ms.append({"call_ms_sorted": sorted(round(t * 1e3, 3) for t in times),
                         "device_ms_median": statistics.median(devs),
                         "upload_ms_median": statistics.median(up) * 1e3})
        return d.sum(em_n) / d.max(sum(times)), r

    e2e_value, _ = e2e_leg(E.TRACE_NONE)
    # full trace (every MAP iteration's hood energies + flags, optimize.cpp:53-58)
    # streamed into caller-owned pinned buffers
    sink = E.TraceSink.pinned(c["em"], MAP_ITERS, H, torch)
    full_value, rf = e2e_leg(E.TRACE_FULL, sink, n=max(3, args.steps // 2))
    trace_d2h = rf.stats["map_iters_total"] * rf.stats["series"] * 9
    full_rec = {"value": full_value, "unit": "EM-iterations/s", "h2d_bytes_per_step": h2d,
                **calls_ms[1],
                "d2h_bytes_per_step": d2h + trace_d2h + 24 * M * c["em"],
                "trace": "full (every MAP iteration's H hood energies f64 + flags u8)",
                "trace_bytes_per_step": trace_d2h}

    # ---- roofline of the dominant kernel (algorithmic bytes) ---------
    vtx_bytes, hood_bytes = map_bytes(R, A, H, S)
    kname = "k_map_fused"
    # fused boundaries: MAP_ITERS + 1 launches per EM move MAP_ITERS x (vertex + hood)
    kbytes = MAP_ITERS * (vtx_bytes + hood_bytes) / (MAP_ITERS + 1)
    kavg = prof["map_loop_ms"] / max(1, prof["map_loop_launches"])
    kernel_split = {"k_map_fused": prof["map_loop_ms"] / prof_steps,
                    "mstep": prof["mstep_ms"] / prof_steps,
                    "mstep_us_per_em": prof["mstep_ms"] * 1e3 / max(1, prof["em_iters"]),
                    "optimize_ms_profiled": prof["optimize_ms"] / prof_steps}
    rl = roofline(kname, kbytes, kavg, ncu_traffic(args.config, kname),
                  note=f"config {args.config}'s per-MAP working set is L2-resident"
                  if args.config in ("A", "B", "C") else "")
    whole = run_bytes(R, A, H, S, c["em"])
    line = {
        "metric": METRIC, "value": value, "unit": "EM-iterations/s", "n_gpus": d.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": c["desc"], "config": args.config,
                   "regions": R, "adjacency": A, "hoods": H, "slots": S, "labels": M,
                   "em_iters_per_step": ems / args.steps, "map_iters_per_step": maps / args.steps,
                   "l2": "flushed between timed steps (256 MiB write)",
                   "parallelism": f"slice-sharded x{d.world} (no data-path collective)",
                   "map_loop": ("active set (extension, --active-set: only items whose inputs "
                                "changed are re-evaluated; identical results, less than the "
                                "reference's per-iteration work)") if act else
                               "dense (every vertex and hood, every MAP iteration)",
                   "structure": (f"packed (adjacency x{r.stats['packed_layout'] // 100}, "
                                 f"hood x{r.stats['packed_layout'] % 100})"
                                 if r.stats["packed_layout"] else "csr"),
                   "timing": "CUDA events on the library stream around each optimize(); "
                             "max over ranks"},
        "vertex_label_evals_per_s": d.sum(M * S * maps) / total_dev_s,
        "unique_vertex_label_evals_per_s": d.sum(M * R * maps) / total_dev_s,
        "kernel_ms_per_step": kernel_split,
        "roofline": rl,
        "whole_step_hbm_frac": (whole / (ms_per_step * 1e-3) / 1e9 / rl["peak"]) if fixed else None,
        "e2e": {"value": e2e_value, "unit": "EM-iterations/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, **calls_ms[0],
                "warmup": f"untimed: >= {args.warmup} calls and >= {E2E_WARM_S} s of calls"},
        "e2e_full_trace": full_rec,
        "gpu_launches": launches,
        "clocks": clocks,
        "setup": {"device_input_build_s": build_inputs_s, "host_ties": info["host_ties"],
                  "note": "phantom -> corrupt -> oversegment -> graph -> cliques -> hoods "
                          "on the device (csrc/synth.cu, structure.cu, hoods.cu)"},
    }
    if M == 2 and not act and not getattr(args, "no_active_record", False):
        # the active-set MAP loop (extension): same labels / parameters, only
        # the items whose inputs changed re-evaluated -- reported beside the
        # headline, never as it (less than the reference's per-iteration work)
        dev_a, em_a = [], 0
        for _ in range(args.warmup):
            ctx.optimize(cfg, fixed_work=fixed, multilabel=ml, trace_level=E.TRACE_NONE,
                         labels_out=labels_out, active_set=True)
        d.barrier()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            ra = ctx.optimize(cfg, fixed_work=fixed, multilabel=ml, trace_level=E.TRACE_NONE,
                              labels_out=labels_out, active_set=True)
            dev_a.append(ra.stats["optimize_ms"])
            em_a += ra.stats["em_iters"]
        d.barrier()
        ra = ctx.optimize(cfg, fixed_work=fixed, multilabel=ml, trace_level=E.TRACE_EM,
                          active_set=True)
        rd = ctx.optimize(cfg, fixed_work=fixed, multilabel=ml, trace_level=E.TRACE_EM)
        same_result = (np.array_equal(ra.labels, rd.labels) and np.array_equal(ra.mu, rd.mu)
                       and np.array_equal(ra.sigma, rd.sigma) and
                       [e.total_energy for e in ra.trace] == [e.total_energy for e in rd.trace])
        act = True
        e2e_a, _ = e2e_leg(E.TRACE_NONE, n=3)
        act = False
        line["active_set"] = {
            "value": d.sum(em_a) / d.max(sum(dev_a) / 1e3), "unit": "EM-iterations/s",
            "e2e": e2e_a, "engaged": bool(ra.stats["active_set"]),
            "bit_identical_to_dense": bool(same_result),
            "note": "extension (DPMRF_RUN_ACTIVE_SET): from the second EM iteration on, only "
                    "vertices whose neighbors' labels changed and hoods whose members' minima "
                    "changed are re-evaluated; same results, less than the reference's "
                    "per-iteration work -- not the headline"}
    if M == 2:
        # segmentation quality of the timed result (not timed): the segment
        # write-back against the phantom truth, on the device
        _, cc = ctx.segment_mask(r.labels, r.mu, mask=False)
        mt = E.compute_metrics(cc)
        line["quality"] = {"precision": mt.precision, "recall": mt.recall,
                           "accuracy": mt.accuracy,
                           "source": "device segment write-back (main.cpp:157-165) vs the "
                                     "phantom truth, confusion on the device; not timed"}
    ctx.close()
    if d.rank == 0 and not args.no_cpu_baseline:
        try:
            v, det = reference_sample(args.config, seconds_budget=args.cpu_seconds, rank_seed=seed)
            line["cpu_baseline"] = {"value": v, "unit": "EM-iterations/s", "cores": det["cores"],
                                    "kind": det["kind"], "sample": det["sample"],
                                    "nproc": det["nproc"], "cpu_model": det["cpu_model"]}
        except Exception as ex:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    return line


# ---- config E: 64-slice stack, slices dealt round-robin to ranks ---------------------------
def run_stack(args, E, torch, d: Dist, cpu=True):
    """Each rank owns slices z = rank, rank+N, ... (seed 42+z); every slice has
    its own context (stream + resident graph/hoods in HBM); a pool of host
    threads drives them concurrently so one slice's host round trip overlaps
    the others' kernels.  A step optimizes all of the rank's slices."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_1809_05018_b200.parallel import shard_slices
    c = CONFIGS["E"]
    zs = shard_slices(args.slices, d.world, d.rank)
    t0 = time.perf_counter()
    ctxs, cfgs, dims = [], [], []
    for z in zs:  # every slice built on the device, resident in its own context
        ctx = E.Context(d.local)
        info = ctx.synthetic_slice(c["size"], c["block"], seed=42 + z)
        ctxs.append(ctx)
        cfgs.append(E.OptimizerConfig(em_max_iters=c["em"], map_max_iters=MAP_ITERS,
                                      rng_seed=42 + z))
        dims.append((ctx.R, info["adjacency"], ctx.H, ctx.S))
    build_s = time.perf_counter() - t0
    workers = min(args.stack_threads, len(ctxs)) or 1

    def run_one(i):
        return ctxs[i].optimize(cfgs[i], fixed_work=True, trace_level=E.TRACE_NONE)

    pool = ThreadPoolExecutor(max_workers=workers)  # (threads started once, not per step)

    def step():
        return list(pool.map(run_one, range(len(ctxs))))

    for _ in range(args.warmup):
        step()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    sampler = ClockSampler(d.local)
    sampler.start()
    times, launches = [], 0
    for _ in range(args.steps):
        flush.zero_()
        d.barrier()
        t0 = time.perf_counter()
        rs = step()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        launches += sum(r.stats["kernel_launches"] for r in rs)
    d.barrier()
    clocks = sampler.stop()
    tot = d.max(sum(times))
    em_total = d.sum(len(ctxs) * c["em"] * args.steps)
    S_tot = d.sum(sum(x[3] for x in dims))
    R_tot = d.sum(sum(x[0] for x in dims))
    # per-GPU roofline: the algorithmic bytes of this rank's slices over its time
    my_bytes = sum(run_bytes(*x, c["em"]) for x in dims) * args.steps
    hbm, peak_kind = peaks()
    ach = d.max(my_bytes) / tot / 1e9
    rec = {
        "value": em_total / tot, "unit": "EM-iterations/s", "n_gpus": d.world,
        "scaling": "strong", "ms_per_step": tot * 1e3 / args.steps,
        "config": {"workload": c["desc"].replace("64", str(args.slices), 1),
                   "slices": args.slices, "slices_per_rank_max": len(ctxs),
                   "host_threads_per_rank": workers,
                   "l2": "flushed between timed steps (256 MiB write)",
                   "timing": "host wall clock around each step (all slices), device "
                             "synchronized; max over ranks"},
        "slices_per_s": args.slices * args.steps / tot,
        "vertex_label_evals_per_s": 2 * S_tot * c["em"] * MAP_ITERS * args.steps / tot,
        "unique_vertex_label_evals_per_s": 2 * R_tot * c["em"] * MAP_ITERS * args.steps / tot,
        "roofline": {"bound": "hbm", "kernel": "whole step (all kernels, per GPU)",
                     "achieved": ach, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": ach / hbm, "traffic": None,
                     "note": "algorithmic bytes (SURVEY §8(d)) of the busiest rank's slices / "
                             "the step time"},
        "gpu_launches": launches, "clocks": clocks,
        "setup": {"device_input_build_s": build_s},
    }
    pool.shutdown()
    for ctx in ctxs:
        ctx.close()
    if cpu and d.rank == 0 and not args.no_cpu_baseline:
        try:
            v, det = reference_sample_stack(args.slices, seconds_budget=min(args.cpu_seconds, 8))
            rec["cpu_baseline"] = {"value": v, "unit": "EM-iterations/s", **det}
        except Exception as ex:  # pragma: no cover
            rec["cpu_baseline"] = {"value": None, "error": str(ex)}
    return rec


# ---- config D: one giant slice partitioned by vertex range across the ranks ----------------
def run_partitioned(args, E, torch, d: Dist, cpu=True, verify=True):
    """Every rank holds the 16384^2 structure in HBM, owns a contiguous vertex
    range and the hoods that follow it (csrc/partition.cu).  Per MAP iteration
    the ranks exchange label and minima halos (grouped ncclSend/Recv); per EM
    iteration they allgather labels + leaf partials.  Total work is fixed:
    "strong" scaling.  With verify, rank 0 also runs the one-device optimize of
    the same slice and the partitioned result must equal it bit for bit."""
    c = CONFIGS["D"]
    seed = 42
    t0 = time.perf_counter()
    ctx = E.Context(d.local)
    info = ctx.synthetic_slice(c["size"], c["block"], brick=c["brick"], seed=seed)
    build_inputs_s = time.perf_counter() - t0
    R, A = info["regions"], info["adjacency"]
    hoods = ctx.get_hoods()
    H, S = hoods.size(), hoods.total_slots()
    nccl = d.world > 1 and not d.shared
    if nccl:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if d.rank == 0:
            uid.copy_(torch.frombuffer(bytearray(E.nccl_unique_id()), dtype=torch.uint8))
        d.dist.broadcast(uid, 0)
        group = E.PartitionGroup.nccl(ctx, bytes(uid.cpu().numpy().tobytes()), d.rank, d.world)
        parts = d.world
    else:
        parts = max(args.local_parts, d.world)
        group = E.PartitionGroup.local(ctx, parts)
    ginfo = group.info()
    cfg = E.OptimizerConfig(num_labels=c["M"], em_max_iters=c["em"], map_max_iters=MAP_ITERS,
                            rng_seed=seed)
    labels_out = np.zeros(R, np.uint32)

    def step():
        return group.optimize(cfg, fixed_work=True, trace_level=E.TRACE_NONE,
                              labels_out=labels_out)

    for _ in range(args.warmup):
        r = step()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    sampler = ClockSampler(d.local)
    sampler.start()
    dev_ms, launches = [], 0
    for _ in range(args.steps):
        flush.zero_()
        d.barrier()
        r = step()
        dev_ms.append(r.stats["optimize_ms"])
        launches += r.stats["kernel_launches"]
    d.barrier()
    clocks = sampler.stop()
    total_dev_s = d.max(sum(dev_ms) / 1e3)
    map_per_step = c["em"] * MAP_ITERS
    exact = None
    if verify:
        one = ctx.optimize(cfg, fixed_work=True, trace_level=E.TRACE_NONE)
        ok = bool(np.array_equal(one.labels, r.labels) and np.array_equal(one.mu, r.mu)
                  and np.array_equal(one.sigma, r.sigma))
        exact = d.sum(0.0 if ok else 1.0) == 0.0
    hbm, peak_kind = peaks()
    ach = run_bytes(R, A, H, S, c["em"]) * args.steps / total_dev_s / 1e9 / (parts if nccl else 1)
    rec = {
        "value": c["em"] * args.steps / total_dev_s, "unit": "EM-iterations/s",
        "n_gpus": d.world, "scaling": "strong", "ms_per_step": total_dev_s * 1e3 / args.steps,
        "config": {"workload": c["desc"] + f"; partitioned by vertex range into {parts} parts",
                   "regions": R, "adjacency": A, "hoods": H, "slots": S, "labels": c["M"],
                   "partitions": parts,
                   "transport": "nccl (grouped send/recv halos, allreduce counters, allgather "
                                "per EM)" if nccl else
                                "local (all partitions on one device, device-copy halos)",
                   "halo_bytes_per_map_rank0": ginfo["halo_bytes_per_map"],
                   "gather_bytes_per_em_rank0": ginfo["gather_bytes_per_em"],
                   "l2": "flushed between timed steps (256 MiB write)",
                   "timing": "CUDA events on the library stream around each optimize(); "
                             "max over ranks"},
        "bit_exact_vs_one_device": exact,
        "vertex_label_evals_per_s": c["M"] * S * map_per_step * args.steps / total_dev_s,
        "unique_vertex_label_evals_per_s": c["M"] * R * map_per_step * args.steps / total_dev_s,
        "roofline": {"bound": "hbm", "kernel": "whole step (all kernels, per GPU)",
                     "achieved": ach, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": ach / hbm, "traffic": None,
                     "note": "algorithmic bytes of the whole fixed-work run (SURVEY §8(d)) / "
                             "time / GPUs"},
        "gpu_launches": launches, "clocks": clocks,
        "setup": {"device_input_build_s": build_inputs_s},
    }
    if cpu and d.rank == 0 and not args.no_cpu_baseline:
        try:
            v, det = reference_sample_arrays(ctx.get_graph(sizes=False), hoods, c["M"])
            rec["cpu_baseline"] = {"value": v, "unit": "EM-iterations/s", **det}
        except Exception as ex:  # pragma: no cover
            rec["cpu_baseline"] = {"value": None, "error": str(ex)}
    group.close()
    ctx.close()
    return rec


def spawn(args):
    """--gpus N without WORLD_SIZE: re-launch as N ranks, one process per GPU."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---- our arm ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="B", choices=sorted(CONFIGS))
    ap.add_argument("--slices", type=int, default=64, help="config E stack depth")
    ap.add_argument("--stack-threads", type=int, default=8)
    ap.add_argument("--local-parts", type=int, default=1,
                    help="config D on one GPU: K vertex-range partitions in one context "
                         "(the multi-GPU schedule with device-copy halos)")
    ap.add_argument("--no-sub-records", action="store_true",
                    help="N>1: skip the stack_E / partitioned_D sub-records")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-active-record", action="store_true",
                    help="skip the active_set sub-record of the slice configs")
    ap.add_argument("--active-set", action="store_true",
                    help="the active-set MAP loop (extension, DPMRF_RUN_ACTIVE_SET): same "
                         "results, re-evaluates only what changed -- not the reference's "
                         "per-iteration work, so never the headline line")
    args = ap.parse_args()
    if os.environ.get("DPMRF_BENCH_ACTIVE") == "1":  # (tools/ab.sh variants)
        args.active_set = True
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)

    import torch
    import torch.distributed as dist

    from paper_1809_05018_b200 import engine as E
    d = Dist(torch, dist)
    if args.config == "E":
        line = run_stack(args, E, torch, d)
        line.update({"metric": METRIC, "steps": args.steps, "warmup": args.warmup,
                     "higher_is_better": True, "vs_baseline": None, "dtype": "f64",
                     "data": "synthetic", "e2e": None})
    elif args.config == "D" and (d.world > 1 or args.local_parts > 1):
        line = run_partitioned(args, E, torch, d)
        line.update({"metric": METRIC, "steps": args.steps, "warmup": args.warmup,
                     "higher_is_better": True, "vs_baseline": None, "dtype": "f64",
                     "data": "synthetic", "e2e": None})
    else:
        line = run_slice(args, E, torch, d)
        if d.world > 1 and args.config == "B" and not args.no_sub_records:
            line["stack_E"] = run_stack(args, E, torch, d)
            line["partitioned_D"] = run_partitioned(args, E, torch, d)
    if d.rank == 0:
        print(json.dumps(line), flush=True)
    d.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
