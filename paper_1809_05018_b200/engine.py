"""Host-side mirror of the reference's engine interface over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/dpmrf/mrf/engine.hpp (and
graph/neighborhoods.hpp for build_neighborhoods), so code written against the
reference reads the same:

    backend = Backend.cuda(0)
    result = optimize(backend, graph, hoods, OptimizerConfig(rng_seed=42))
    result.labels, result.params.mu, result.params.sigma, result.trace

Every call runs on the B200 through libdpmrf_cuda.so; there is no CPU path.
Errors map to the reference's exception types:
    dpmrf::InputError      -> InputError          (error.hpp:11)
    std::invalid_argument  -> ValueError
    std::out_of_range      -> IndexError
    device failures        -> CudaError
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N

# ---- errors ------------------------------------------------------------------------
DPMRF_OK, DPMRF_INPUT_ERROR, DPMRF_INVALID_ARGUMENT, DPMRF_OUT_OF_RANGE = 0, 1, 2, 3
DPMRF_CUDA_ERROR, DPMRF_NCCL_ERROR, DPMRF_INTERNAL_ERROR = 4, 5, 6

TRACE_NONE, TRACE_EM, TRACE_FULL = 0, 1, 2
RUN_FIXED_WORK, RUN_MULTILABEL, RUN_KERNEL_TIMING, RUN_NO_GRAPH = 1, 2, 4, 16
RUN_HOST_LOG, RUN_CSR, RUN_UNFUSED, RUN_ACTIVE_SET = 128, 256, 512, 1024

K_SIGMA_FLOOR = 1e-3  # kSigmaFloor, model.hpp:9


class InputError(RuntimeError):
    """dpmrf::InputError (proj/include/dpmrf/error.hpp:11)."""


class CudaError(RuntimeError):
    pass


def _check(status: int, where: str):
    if status == DPMRF_OK:
        return
    msg = f"{where}: {N.cuda().dpmrf_last_error().decode(errors='replace')}"
    if status == DPMRF_INPUT_ERROR:
        raise InputError(msg)
    if status == DPMRF_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == DPMRF_OUT_OF_RANGE:
        raise IndexError(msg)
    if status in (DPMRF_CUDA_ERROR, DPMRF_NCCL_ERROR):
        raise CudaError(msg)
    raise RuntimeError(msg)


def _u32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint32))


def _f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


# ---- value types (model.hpp, region_graph.hpp, neighborhoods.hpp) ------------------
@dataclass
class OptimizerConfig:
    """OptimizerConfig, model.hpp:19-27 (same defaults)."""

    num_labels: int = 2
    em_max_iters: int = 20
    map_max_iters: int = 10
    convergence_window: int = 3
    convergence_tol: float = 1e-4
    beta: float = 1.0
    rng_seed: int = 0

    def c(self) -> N.CConfig:
        return N.CConfig(self.num_labels, self.em_max_iters, self.map_max_iters,
                         self.convergence_window, self.convergence_tol, self.beta,
                         self.rng_seed & ((1 << 64) - 1))


@dataclass
class LabelParams:
    """LabelParams, model.hpp:12-17."""

    mu: np.ndarray
    sigma: np.ndarray

    def num_labels(self) -> int:
        return len(self.mu)


@dataclass
class RegionGraph:
    """RegionGraph, region_graph.hpp:14-25 (CSR + per-region means)."""

    offsets: np.ndarray
    neighbors: np.ndarray
    region_mean: np.ndarray
    region_size: Optional[np.ndarray] = None

    @property
    def num_vertices(self) -> int:
        return len(self.offsets) - 1

    def degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])


@dataclass
class NeighborhoodSet:
    """NeighborhoodSet, neighborhoods.hpp:15-23."""

    offsets: np.ndarray
    members: np.ndarray
    source_clique: Optional[np.ndarray] = None

    def size(self) -> int:
        return len(self.offsets) - 1

    def total_slots(self) -> int:
        return len(self.members)


@dataclass
class CliqueSet:
    """CliqueSet, cliques.hpp:14-22."""

    offsets: np.ndarray
    members: np.ndarray

    def size(self) -> int:
        return len(self.offsets) - 1


@dataclass
class ReplicatedIndex:
    """ReplicatedIndex, model.hpp:29-37."""

    test_label: np.ndarray
    old_index: np.ndarray
    hood_id: np.ndarray


@dataclass
class MinLabelEnergies:
    """MinLabelEnergies, engine.hpp:48-51."""

    energy: np.ndarray
    label: np.ndarray


@dataclass
class MapIterationLog:
    hood_energy: np.ndarray
    converged: np.ndarray


@dataclass
class EmIterationLog:
    map_iters: List[MapIterationLog]
    total_energy: float
    converged: bool
    params: LabelParams
    num_map_iters: int = 0

    # flat aliases used by the parity helpers
    @property
    def mu(self):
        return self.params.mu

    @property
    def sigma(self):
        return self.params.sigma


@dataclass
class OptimizeResult:
    """OptimizeResult, engine.hpp:87-91 (+ device statistics)."""

    labels: np.ndarray
    params: LabelParams
    trace: List[EmIterationLog] = field(default_factory=list)
    stats: Optional[dict] = None

    @property
    def mu(self):
        return self.params.mu

    @property
    def sigma(self):
        return self.params.sigma


# ---- backend selector (dpp::Backend, backend.hpp:16-35, + a Cuda kind) ----------
@dataclass(frozen=True)
class Backend:
    kind: str = "cuda"
    device: int = 0

    @staticmethod
    def cuda(device: int = 0) -> "Backend":
        return Backend("cuda", device)


# ---- full-trace destination ----------------------------------------------------------
class TraceSink:
    """Caller-owned buffers for the full trace (dpmrf_set_trace_sink): row
    em * map_max_iters + t holds MAP iteration t of EM iteration em (hood
    energies f64 / flags u8, ``stride`` values per row).  ``pinned`` allocates
    page-locked memory (link-rate DMA straight from the device)."""

    def __init__(self, energy: np.ndarray, flags: np.ndarray, rows: int, stride: int):
        assert energy.dtype == np.float64 and flags.dtype == np.uint8
        assert energy.size >= rows * stride and flags.size >= rows * stride
        self.energy, self.flags, self.rows, self.stride = energy, flags, rows, stride
        self.energy_rows = energy[:rows * stride].reshape(rows, stride)
        self.flag_rows = flags[:rows * stride].reshape(rows, stride)

    @classmethod
    def host(cls, em_max_iters: int, map_max_iters: int, num_hoods: int) -> "TraceSink":
        rows, stride = max(1, em_max_iters * map_max_iters), max(1, num_hoods)
        return cls(np.empty(rows * stride), np.empty(rows * stride, np.uint8), rows, stride)

    @classmethod
    def pinned(cls, em_max_iters: int, map_max_iters: int, num_hoods: int, torch) -> "TraceSink":
        rows, stride = max(1, em_max_iters * map_max_iters), max(1, num_hoods)
        e = torch.empty(rows * stride, dtype=torch.float64).pin_memory().numpy()
        f = torch.empty(rows * stride, dtype=torch.uint8).pin_memory().numpy()
        return cls(e, f, rows, stride)

    def fits(self, config, series: int) -> bool:
        return (config is not None and self.rows >= config.em_max_iters * config.map_max_iters
                and self.stride >= series)


# ---- context: resident graph + hoods in HBM ---------------------------------------
class Context:
    """One dpmrf_context: a CUDA stream plus the resident graph and hoods."""

    def __init__(self, device: int = 0):
        self._lib = N.cuda()
        h = ct.c_void_p()
        _check(self._lib.dpmrf_context_create(device, ct.byref(h)), "dpmrf_context_create")
        self.h = h
        self.device = device
        self._graph_key = None
        self._hoods_key = None
        self.R = 0
        self.H = 0
        self.S = 0
        self._cliques_n = (0, 0)
        self._img_n = 0  # pixels of the resident image (make_phantom)
        self._img_regions = 0  # regions of the resident label map (oversegment)
        self._sink = None  # attached TraceSink (dpmrf_set_trace_sink)

    def close(self):
        if self.h:
            self._lib.dpmrf_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- resident inputs --
    def set_graph(self, graph: RegionGraph):
        off, nbr, mean = _u32(graph.offsets), _u32(graph.neighbors), _f64(graph.region_mean)
        R = len(off) - 1
        _check(self._lib.dpmrf_set_graph(self.h, R, N.ptr(off), N.ptr(nbr), N.ptr(mean)),
               "dpmrf_set_graph")
        self.R = R
        self._graph_key = graph

    def set_hoods(self, hoods: NeighborhoodSet):
        off, mem = _u32(hoods.offsets), _u32(hoods.members)
        _check(self._lib.dpmrf_set_hoods(self.h, len(off) - 1, N.ptr(off), N.ptr(mem)),
               "dpmrf_set_hoods")
        self.H, self.S = len(off) - 1, len(mem)
        self._hoods_key = hoods

    def build_neighborhoods(self, cliques: CliqueSet, k: int = 1) -> int:
        off, mem = _u32(cliques.offsets), _u32(cliques.members)
        n = ct.c_uint64(0)
        _check(self._lib.dpmrf_build_neighborhoods(self.h, len(off) - 1, N.ptr(off), N.ptr(mem),
                                                   k, ct.byref(n)), "build_neighborhoods")
        self.H, self.S = len(off) - 1, n.value
        self._hoods_key = None
        return n.value

    def get_hoods(self) -> NeighborhoodSet:
        H, S = ct.c_uint64(0), ct.c_uint64(0)
        _check(self._lib.dpmrf_get_hoods(self.h, ct.byref(H), ct.byref(S), None, None, None),
               "dpmrf_get_hoods")
        off = np.zeros(H.value + 1, np.uint32)
        mem = np.zeros(S.value, np.uint32)
        src = np.zeros(H.value, np.uint32)
        _check(self._lib.dpmrf_get_hoods(self.h, None, None, N.ptr(off), N.ptr(mem), N.ptr(src)),
               "dpmrf_get_hoods")
        return NeighborhoodSet(off, mem, src)

    # -- synthetic inputs on the device --
    def make_phantom(self, width, height, pore_fraction=0.25, sp_rate=0.0, gauss_sigma=0.0,
                     ringing=False, seed=0, copy_out=True):
        """gen_phantom + corrupt (phantom.cpp:54-150) on the device; the image
        stays resident.  Returns (truth, image, host_ties) -- arrays are None
        unless copy_out."""
        spec = N.CPhantomSpec(width, height, pore_fraction, sp_rate, gauss_sigma, int(ringing),
                              seed)
        n = width * height
        truth = np.zeros(n, np.uint8) if copy_out else None
        image = np.zeros(n, np.uint8) if copy_out else None
        ties = ct.c_uint32(0)
        _check(self._lib.dpmrf_make_phantom(self.h, ct.byref(spec), N.ptr(truth), N.ptr(image),
                                            ct.byref(ties)), "make_phantom")
        self._img_n = n
        return truth, image, ties.value

    def oversegment(self, block: int, brick: bool = False, copy_out=True):
        """Grid (label_map.cpp:79-94) or brick oversegmentation of the resident
        image on the device -> (num_regions, region map or None)."""
        R = ct.c_uint32(0)
        region = np.zeros(self._img_n, np.uint32) if copy_out and self._img_n else None
        _check(self._lib.dpmrf_oversegment(self.h, block, int(brick), ct.byref(R), N.ptr(region)),
               "oversegment")
        self._img_regions = R.value
        return R.value, region

    def build_region_graph_resident(self) -> int:
        A = ct.c_uint64(0)
        _check(self._lib.dpmrf_build_region_graph_resident(self.h, ct.byref(A)),
               "build_region_graph_resident")
        self.R = self._img_regions  # (the graph's vertices are the map's regions)
        self._graph_key = None
        self._hoods_key = None
        return A.value

    def synthetic_slice(self, size=2560, block=8, brick=False, seed=42, pore=0.25, sp=0.05,
                        gauss=100.0, ringing=True, height=None) -> dict:
        """The BASELINE.json synthetic slice built entirely on the device:
        phantom -> corrupt -> oversegment -> region graph -> maximal cliques
        -> neighborhoods, all resident (ready for optimize)."""
        h = height or size
        _, _, ties = self.make_phantom(size, h, pore, sp, gauss, ringing, seed, copy_out=False)
        R, _ = self.oversegment(block, brick, copy_out=False)
        A = self.build_region_graph_resident()
        self.R = R
        C, CS = self.enumerate_maximal_cliques()
        S = self.build_neighborhoods_resident()
        return {"regions": R, "adjacency": A, "cliques": C, "slots": S, "host_ties": ties}

    def validate_label_map(self, width: int, height: int, region) -> int:
        """validate_label_map (label_map.cpp:38-78) on the device -> num_regions;
        InputError with the reference's message otherwise."""
        reg = np.ascontiguousarray(region, np.uint32)
        if reg.size != width * height:
            raise InputError("label map: size does not match dimensions")
        num = ct.c_uint32(0)
        _check(self._lib.dpmrf_validate_label_map(self.h, width, height, N.ptr(reg),
                                                  ct.byref(num)), "validate_label_map")
        return num.value

    # -- evaluation on the device --
    def confusion(self, pred, truth) -> "ConfusionCounts":
        """confusion_u8 (metrics.cpp:8-14, scalar_kernels.cpp:48-63) of two
        equally long u8 arrays (nonzero = positive) on the device."""
        a, b = np.ascontiguousarray(pred, np.uint8), np.ascontiguousarray(truth, np.uint8)
        if a.size != b.size:
            raise InputError("confusion: image dimensions differ")
        c = np.zeros(4, np.uint64)
        _check(self._lib.dpmrf_confusion(self.h, a.size, N.ptr(a), N.ptr(b), N.ptr(c)),
               "confusion")
        return ConfusionCounts(*(int(x) for x in c))

    def segment_mask(self, labels, mu, *, mask=True, counts=True):
        """The segment write-back (main.cpp:157-165): mask[p] =
        labels[region[p]] == pore (the darker class) over the resident label
        map, and its confusion against the resident phantom truth.  Returns
        (mask or None, ConfusionCounts or None)."""
        lab = np.ascontiguousarray(labels, np.uint32)
        m = np.asarray(mu, np.float64)
        out = np.zeros(self._img_n, np.uint8) if mask else None
        c = np.zeros(4, np.uint64) if counts else None
        _check(self._lib.dpmrf_segment_mask(self.h, lab.size, N.ptr(lab), N.ptr(m), N.ptr(out),
                                            N.ptr(c)), "segment_mask")
        return out, (ConfusionCounts(*(int(x) for x in c)) if counts else None)

    # -- device structure builders --
    def build_region_graph(self, width: int, height: int, pixels, region, num_regions: int) -> int:
        """build_region_graph (region_graph.cpp:10-73) on the device from a u8
        image and a validated u32 label map; the graph becomes resident.
        Returns the adjacency length A."""
        px = np.ascontiguousarray(pixels, np.uint8).reshape(-1)
        reg = _u32(np.asarray(region).reshape(-1))
        if len(px) != width * height or len(reg) != width * height:
            raise InputError("region graph: image and label map dimensions differ")
        A = ct.c_uint64(0)
        _check(self._lib.dpmrf_build_region_graph(self.h, width, height, N.ptr(px), N.ptr(reg),
                                                  num_regions, ct.byref(A)), "build_region_graph")
        self.R = num_regions
        self._img_n, self._img_regions = width * height, num_regions
        self._graph_key = None
        self._hoods_key = None
        return A.value

    def build_region_graph_device(self, width: int, height: int, pixels_ptr: int,
                                  region_ptr: int, num_regions: int) -> int:
        """build_region_graph from device-resident u8 pixels / u32 region ids
        (raw device pointers, e.g. torch tensors' data_ptr())."""
        A = ct.c_uint64(0)
        _check(self._lib.dpmrf_build_region_graph_device(self.h, width, height, pixels_ptr,
                                                         region_ptr, num_regions, ct.byref(A)),
               "build_region_graph_device")
        self.R = num_regions
        self._graph_key = None
        self._hoods_key = None
        return A.value

    def get_graph(self, sizes: bool = True) -> RegionGraph:
        R, A = ct.c_uint32(0), ct.c_uint64(0)
        _check(self._lib.dpmrf_get_graph(self.h, ct.byref(R), ct.byref(A), None, None, None, None),
               "get_graph")
        off = np.zeros(R.value + 1, np.uint32)
        nbr = np.zeros(A.value, np.uint32)
        mean = np.zeros(R.value)
        size = np.zeros(R.value, np.uint32) if sizes else None
        _check(self._lib.dpmrf_get_graph(self.h, None, None, N.ptr(off), N.ptr(nbr), N.ptr(mean),
                                         N.ptr(size) if sizes else None), "get_graph")
        return RegionGraph(off, nbr, mean, size)

    def enumerate_maximal_cliques(self):
        """enumerate_maximal_cliques (cliques.cpp:53-106) on the device over the
        resident graph; the cliques stay resident.  Returns (C, members)."""
        C, CS = ct.c_uint64(0), ct.c_uint64(0)
        _check(self._lib.dpmrf_enumerate_maximal_cliques(self.h, ct.byref(C), ct.byref(CS)),
               "enumerate_maximal_cliques")
        self._cliques_n = (C.value, CS.value)
        return C.value, CS.value

    def get_cliques(self) -> CliqueSet:
        C, CS = self._cliques_n
        off = np.zeros(C + 1, np.uint32)
        mem = np.zeros(CS, np.uint32)
        _check(self._lib.dpmrf_get_cliques(self.h, N.ptr(off), N.ptr(mem)), "get_cliques")
        return CliqueSet(off, mem)

    def build_neighborhoods_resident(self, k: int = 1) -> int:
        n = ct.c_uint64(0)
        _check(self._lib.dpmrf_build_neighborhoods_resident(self.h, k, ct.byref(n)),
               "build_neighborhoods_resident")
        self.H, self.S = self._cliques_n[0], n.value
        self._hoods_key = None
        return n.value

    # -- the optimization phase --
    def optimize(self, config: OptimizerConfig, *, fixed_work=False, multilabel=False,
                 trace_level=TRACE_FULL, kernel_timing=False, labels_out=None,
                 graphs=True, host_log=False, csr=False, fused=True,
                 trace_sink: Optional["TraceSink"] = None,
                 active_set=False) -> OptimizeResult:
        """optimize (optimize.cpp:31-74) on the resident graph + hoods.
        multilabel=True allows num_labels != 2 (extension; the reference's
        validate_config rejects it, optimize.cpp:14).  trace_sink: caller-owned
        (pinned) buffers the full trace is streamed into (dpmrf_set_trace_sink);
        the returned MapIterationLogs are views into it.  active_set=True
        (extension, DPMRF_RUN_ACTIVE_SET): re-evaluate only what changed --
        same results, less than the reference's per-iteration work."""
        M = config.num_labels
        flags = (RUN_FIXED_WORK if fixed_work else 0) | (RUN_MULTILABEL if multilabel else 0) | \
            (RUN_KERNEL_TIMING if kernel_timing else 0) | (RUN_HOST_LOG if host_log else 0) | \
            (RUN_CSR if csr else 0) | (0 if fused else RUN_UNFUSED) | \
            (0 if graphs else RUN_NO_GRAPH) | (RUN_ACTIVE_SET if active_set else 0)
        opts = N.CRunOptions(flags, trace_level)
        cfg = config.c()
        labels = labels_out if labels_out is not None else np.zeros(self.R, np.uint32)
        mu, sigma = np.zeros(M), np.zeros(M)
        self._attach(trace_sink)
        _check(self._lib.dpmrf_optimize(self.h, ct.byref(cfg), ct.byref(opts), N.ptr(labels),
                                        N.ptr(mu), N.ptr(sigma)), "optimize")
        return OptimizeResult(labels, LabelParams(mu, sigma),
                              self._trace(M, trace_level, trace_sink, config), self.stats())

    def _attach(self, sink: Optional["TraceSink"]):
        if sink is None:
            if self._sink is not None:
                _check(self._lib.dpmrf_set_trace_sink(self.h, None, None, 0, 0), "trace_sink")
                self._sink = None
            return
        if sink is not self._sink:
            _check(self._lib.dpmrf_set_trace_sink(self.h, N.ptr(sink.energy), N.ptr(sink.flags),
                                                  sink.rows, sink.stride), "trace_sink")
            self._sink = sink

    def optimize_arrays(self, graph: RegionGraph, hoods: NeighborhoodSet,
                        config: OptimizerConfig, *, fixed_work=False, multilabel=False,
                        trace_level=TRACE_FULL, labels_out=None,
                        trace_sink: Optional["TraceSink"] = None,
                        active_set=False) -> OptimizeResult:
        """optimize(backend, graph, hoods, config) in ONE C-ABI call
        (dpmrf_optimize_arrays): host arrays in, labels / params out."""
        M = config.num_labels
        self._attach(trace_sink)
        flags = (RUN_FIXED_WORK if fixed_work else 0) | (RUN_MULTILABEL if multilabel else 0) | \
            (RUN_ACTIVE_SET if active_set else 0)
        opts = N.CRunOptions(flags, trace_level)
        cfg = config.c()
        off, nbr, mean = _u32(graph.offsets), _u32(graph.neighbors), _f64(graph.region_mean)
        hoff, hmem = _u32(hoods.offsets), _u32(hoods.members)
        R = len(off) - 1
        labels = labels_out if labels_out is not None else np.zeros(R, np.uint32)
        mu, sigma = np.zeros(M), np.zeros(M)
        _check(self._lib.dpmrf_optimize_arrays(self.h, R, N.ptr(off), N.ptr(nbr), N.ptr(mean),
                                               len(hoff) - 1, N.ptr(hoff), N.ptr(hmem),
                                               ct.byref(cfg), ct.byref(opts), N.ptr(labels),
                                               N.ptr(mu), N.ptr(sigma)), "optimize_arrays")
        self.R, self.H, self.S = R, len(hoff) - 1, len(hmem)
        return OptimizeResult(labels, LabelParams(mu, sigma),
                              self._trace(M, trace_level, trace_sink, config), self.stats())

    def _trace(self, M, level, sink=None, config=None) -> List[EmIterationLog]:
        if level == TRACE_NONE:
            return []
        em_n, series = ct.c_int32(0), ct.c_uint64(0)
        _check(self._lib.dpmrf_trace_info(self.h, ct.byref(em_n), ct.byref(series)), "trace")
        on_device = sink is not None and self.stats()["device_loop"] == 1  # rows in the sink
        out = []
        for em in range(em_n.value):
            it, tot, conv = ct.c_int32(0), ct.c_double(0), ct.c_uint8(0)
            mu, sg = np.zeros(M), np.zeros(M)
            _check(self._lib.dpmrf_trace_em(self.h, em, ct.byref(it), ct.byref(tot),
                                            ct.byref(conv), N.ptr(mu), N.ptr(sg)), "trace_em")
            maps = []
            if level >= TRACE_FULL and sink is not None and on_device and \
                    sink.fits(config, series.value):
                for t in range(it.value):
                    row = em * config.map_max_iters + t
                    maps.append(MapIterationLog(sink.energy_rows[row, :series.value],
                                                sink.flag_rows[row, :series.value]))
            elif level >= TRACE_FULL:
                for t in range(it.value):
                    e = np.zeros(series.value)
                    f = np.zeros(series.value, np.uint8)
                    _check(self._lib.dpmrf_trace_map(self.h, em, t, N.ptr(e), N.ptr(f)),
                           "trace_map")
                    maps.append(MapIterationLog(e, f))
            out.append(EmIterationLog(maps, tot.value, bool(conv.value), LabelParams(mu, sg),
                                      it.value))
        return out

    def debug_log(self, x):
        """The device's correctly rounded log (used for log(sigma) on the device loop)."""
        x = _f64(x)
        out = np.zeros(len(x))
        _check(self._lib.dpmrf_debug_log(self.h, len(x), N.ptr(x), N.ptr(out)), "debug_log")
        return out

    def stats(self) -> dict:
        s = N.CRunStats()
        _check(self._lib.dpmrf_get_stats(self.h, ct.byref(s)), "get_stats")
        return {k: getattr(s, k) for k, _ in N.CRunStats._fields_}

    # -- step functions (engine.hpp) on the resident structures --
    def replicate_by_label(self, M) -> ReplicatedIndex:
        E = M * self.S
        tl, oi, hid = (np.zeros(E, np.uint32) for _ in range(3))
        _check(self._lib.dpmrf_replicate_by_label(self.h, M, N.ptr(tl), N.ptr(oi), N.ptr(hid)),
               "replicate_by_label")
        return ReplicatedIndex(tl, oi, hid)

    def slot_hood_map(self):
        out = np.zeros(self.S, np.uint32)
        _check(self._lib.dpmrf_slot_hood_map(self.h, N.ptr(out)), "slot_hood_map")
        return out

    def discord_counts(self, labels, M):
        lab = _u32(labels)
        out = np.zeros(M * self.R, np.uint32)
        _check(self._lib.dpmrf_discord_counts(self.h, N.ptr(lab), M, N.ptr(out)), "discord_counts")
        return out

    def compute_energies(self, rep: ReplicatedIndex, params: LabelParams, labels, beta):
        tl, oi = _u32(rep.test_label), _u32(rep.old_index)
        mu, sg, lab = _f64(params.mu), _f64(params.sigma), _u32(labels)
        out = np.zeros(len(tl))
        _check(self._lib.dpmrf_compute_energies(self.h, len(tl), N.ptr(tl), N.ptr(oi), len(mu),
                                                N.ptr(mu), N.ptr(sg), N.ptr(lab), beta,
                                                N.ptr(out)), "compute_energies")
        return out

    def min_label_energies(self, rep: ReplicatedIndex, energies, num_slots) -> MinLabelEnergies:
        tl, oi, en = _u32(rep.test_label), _u32(rep.old_index), _f64(energies)
        if len(tl) != len(en) or len(oi) != len(en):
            raise ValueError("min_label_energies: replicated index/energies mismatch")
        oe, ol = np.zeros(num_slots), np.zeros(num_slots, np.uint32)
        _check(self._lib.dpmrf_min_label_energies(self.h, len(en), N.ptr(tl), N.ptr(oi),
                                                  N.ptr(en), num_slots, N.ptr(oe), N.ptr(ol)),
               "min_label_energies")
        return MinLabelEnergies(oe, ol)

    def neighborhood_energy_sums(self, slot_hood, min_energy):
        k, x = _u32(slot_hood), _f64(min_energy)
        if len(k) != len(x):
            raise ValueError("reduce_by_key: keys/values length mismatch")
        out = np.zeros(max(len(k), 1))
        n = ct.c_uint64(0)
        _check(self._lib.dpmrf_neighborhood_energy_sums(self.h, len(k), N.ptr(k), N.ptr(x),
                                                        N.ptr(out), ct.byref(n)),
               "neighborhood_energy_sums")
        return out[:n.value].copy()

    def check_convergence(self, history, window, tol):
        if len(history) == 0:
            return np.zeros(0, np.uint8)
        h = _f64(np.asarray(history, dtype=np.float64).reshape(len(history), -1))
        out = np.zeros(h.shape[1], np.uint8)
        _check(self._lib.dpmrf_check_convergence(self.h, h.shape[0], h.shape[1], N.ptr(h), window,
                                                 tol, N.ptr(out)), "check_convergence")
        return out

    def update_labels(self, argmin_label, old_labels):
        a, old = _u32(argmin_label), _u32(old_labels)
        if len(a) != self.S:
            raise ValueError("update_labels: one argmin per hood slot required")
        out = np.zeros(len(old), np.uint32)
        _check(self._lib.dpmrf_update_labels(self.h, N.ptr(a), len(old), N.ptr(old), N.ptr(out)),
               "update_labels")
        return out

    def update_parameters(self, labels, previous: LabelParams) -> LabelParams:
        lab = _u32(labels)
        if len(lab) != self.R:
            raise ValueError("update_parameters: one label per vertex required")
        M = len(previous.mu)
        mu, sg = np.zeros(M), np.zeros(M)
        _check(self._lib.dpmrf_update_parameters(self.h, N.ptr(lab), M, N.ptr(_f64(previous.mu)),
                                                 N.ptr(_f64(previous.sigma)), N.ptr(mu),
                                                 N.ptr(sg)), "update_parameters")
        return LabelParams(mu, sg)

    def init_random(self, num_labels, num_vertices, seed, allow_multilabel=False):
        mu, sg = np.zeros(num_labels), np.zeros(num_labels)
        lab = np.zeros(num_vertices, np.uint32)
        _check(self._lib.dpmrf_init_random(self.h, num_labels, num_vertices,
                                           seed & ((1 << 64) - 1), int(allow_multilabel),
                                           N.ptr(mu), N.ptr(sg), N.ptr(lab)), "init_random")
        return LabelParams(mu, sg), lab


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it and ships it to the others)."""
    buf = (ct.c_uint8 * 128)()
    _check(N.cuda().dpmrf_nccl_unique_id(buf), "nccl_unique_id")
    return bytes(buf)


class PartitionGroup:
    """Vertex-range partitioned optimize of ONE region graph (config D).

    ``PartitionGroup.local(ctx, world)`` runs every partition inside ``ctx`` on
    one device (halos by device copies); ``PartitionGroup.nccl(ctx, uid, rank,
    world)`` is one rank of a one-process-per-GPU NCCL group.  ``optimize``
    returns exactly what ``Context.optimize`` returns on one device."""

    def __init__(self, ctx: Context, handle, world: int, rank: int):
        self.ctx, self.h, self.world, self.rank = ctx, handle, world, rank
        self._lib = N.cuda()

    @classmethod
    def local(cls, ctx: Context, world: int) -> "PartitionGroup":
        h = ct.c_void_p()
        _check(N.cuda().dpmrf_group_create_local(ctx.h, world, ct.byref(h)), "group_create_local")
        return cls(ctx, h, world, -1)

    @classmethod
    def nccl(cls, ctx: Context, uid: bytes, rank: int, world: int) -> "PartitionGroup":
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        h = ct.c_void_p()
        buf = (ct.c_uint8 * 128).from_buffer_copy(uid)
        _check(N.cuda().dpmrf_group_create_nccl(ctx.h, buf, rank, world, ct.byref(h)),
               "group_create_nccl")
        return cls(ctx, h, world, rank)

    def close(self):
        if self.h:
            self._lib.dpmrf_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = N.CGroupInfo()
        _check(self._lib.dpmrf_group_info_get(self.h, ct.byref(i)), "group_info")
        return {k: getattr(i, k) for k, _ in N.CGroupInfo._fields_}

    def optimize(self, config: OptimizerConfig, *, fixed_work=False, multilabel=False,
                 trace_level=TRACE_EM, host_log=False, csr=False, graphs=True,
                 labels_out=None) -> OptimizeResult:
        M = config.num_labels
        flags = (RUN_FIXED_WORK if fixed_work else 0) | (RUN_MULTILABEL if multilabel else 0) | \
            (RUN_HOST_LOG if host_log else 0) | (RUN_CSR if csr else 0) | \
            (0 if graphs else RUN_NO_GRAPH)
        opts = N.CRunOptions(flags, trace_level)
        cfg = config.c()
        labels = labels_out if labels_out is not None else np.zeros(self.ctx.R, np.uint32)
        mu, sigma = np.zeros(M), np.zeros(M)
        _check(self._lib.dpmrf_optimize_partitioned(self.h, ct.byref(cfg), ct.byref(opts),
                                                    N.ptr(labels), N.ptr(mu), N.ptr(sigma)),
               "optimize_partitioned")
        return OptimizeResult(labels, LabelParams(mu, sigma), self.ctx._trace(M, trace_level),
                              self.ctx.stats())


# ---- free functions with the reference's signatures --------------------------------
_contexts = {}


def context_for(backend: Backend) -> Context:
    if backend.kind != "cuda":
        raise InputError(f"unsupported backend kind {backend.kind!r} (this build is CUDA-only)")
    ctx = _contexts.get(backend.device)
    if ctx is None:
        ctx = _contexts[backend.device] = Context(backend.device)
    return ctx


def _resident(ctx: Context, graph: RegionGraph, hoods: Optional[NeighborhoodSet] = None):
    """The reference reads its inputs by const& on every call, so the free
    functions upload them on every call (a caller may mutate the arrays
    between calls); keep them resident with an explicit Context instead."""
    ctx.set_graph(graph)
    if hoods is not None:
        ctx.set_hoods(hoods)


def optimize(backend: Backend, graph: RegionGraph, hoods: NeighborhoodSet,
             config: OptimizerConfig, **kw) -> OptimizeResult:
    """optimize, engine.hpp:99-100 / optimize.cpp:31-74."""
    ctx = context_for(backend)
    _resident(ctx, graph, hoods)
    return ctx.optimize(config, **kw)


def build_region_graph(backend: Backend, width: int, height: int, pixels, region,
                       num_regions: int) -> RegionGraph:
    """build_region_graph, region_graph.hpp:31-33 (GrayImage + LabelMap as arrays), on the device."""
    ctx = context_for(backend)
    ctx.build_region_graph(width, height, pixels, region, num_regions)
    g = ctx.get_graph()
    ctx._graph_key = g
    return g


def enumerate_maximal_cliques(backend: Backend, graph: RegionGraph) -> CliqueSet:
    """enumerate_maximal_cliques, cliques.hpp:24-27 / cliques.cpp:53-106, on the device."""
    ctx = context_for(backend)
    _resident(ctx, graph)
    ctx.enumerate_maximal_cliques()
    return ctx.get_cliques()


def build_neighborhoods(backend: Backend, graph: RegionGraph, cliques: CliqueSet,
                        k: int = 1) -> NeighborhoodSet:
    """build_neighborhoods, neighborhoods.hpp:28-29 / neighborhoods.cpp:10-57 (on the device)."""
    ctx = context_for(backend)
    _resident(ctx, graph)
    ctx.build_neighborhoods(cliques, k)
    return ctx.get_hoods()


def init_random(num_labels, num_vertices, seed, backend: Backend = Backend.cuda()):
    """init_random, engine.hpp:20-21 -> (LabelParams, labels)."""
    return context_for(backend).init_random(num_labels, num_vertices, seed)


def replicate_by_label(backend: Backend, hoods: NeighborhoodSet, num_labels) -> ReplicatedIndex:
    ctx = context_for(backend)
    ctx.set_hoods(hoods)
    return ctx.replicate_by_label(num_labels)


def slot_hood_map(backend: Backend, hoods: NeighborhoodSet):
    ctx = context_for(backend)
    ctx.set_hoods(hoods)
    return ctx.slot_hood_map()


def discord_counts(backend: Backend, graph: RegionGraph, labels, num_labels):
    ctx = context_for(backend)
    _resident(ctx, graph)
    return ctx.discord_counts(labels, num_labels)


def compute_energies(backend: Backend, graph: RegionGraph, hoods: NeighborhoodSet,
                     rep: ReplicatedIndex, params: LabelParams, labels, beta):
    ctx = context_for(backend)
    _resident(ctx, graph, hoods)
    return ctx.compute_energies(rep, params, labels, beta)


def min_label_energies(backend: Backend, rep: ReplicatedIndex, energies, num_slots):
    return context_for(backend).min_label_energies(rep, energies, num_slots)


def neighborhood_energy_sums(backend: Backend, slot_hood, min_energy):
    return context_for(backend).neighborhood_energy_sums(slot_hood, min_energy)


def check_convergence(backend: Backend, history, window, tol):
    return context_for(backend).check_convergence(history, window, tol)


def update_labels(backend: Backend, hoods: NeighborhoodSet, argmin_label, old_labels):
    ctx = context_for(backend)
    ctx.set_hoods(hoods)
    return ctx.update_labels(argmin_label, old_labels)


def update_parameters(backend: Backend, graph: RegionGraph, labels, previous: LabelParams):
    ctx = context_for(backend)
    _resident(ctx, graph)
    return ctx.update_parameters(labels, previous)


# ---- evaluation (proj/include/dpmrf/eval/metrics.hpp) ------------------------------
@dataclass
class ConfusionCounts:
    """ConfusionCounts, metrics.hpp:9-14 (class 1 / pore positive)."""
    tp: int = 0
    tn: int = 0
    fp: int = 0
    fn: int = 0


@dataclass
class Metrics:
    """Metrics, metrics.hpp:20-26."""
    precision: float = 0.0
    recall: float = 0.0
    accuracy: float = 0.0
    precision_defined: bool = True
    recall_defined: bool = True


@dataclass
class BinaryImage:
    """BinaryImage, image.hpp:22-28: width x height u8 pixels, 1 = pore."""
    width: int
    height: int
    pixels: np.ndarray


def confusion(backend: Backend, pred: BinaryImage, truth: BinaryImage) -> ConfusionCounts:
    """confusion, metrics.hpp:17-18 / metrics.cpp:8-14, counted on the device;
    InputError on a shape mismatch as in the reference."""
    if pred.width != truth.width or pred.height != truth.height:
        raise InputError("confusion: image dimensions differ")
    return context_for(backend).confusion(pred.pixels, truth.pixels)


def compute_metrics(c: ConfusionCounts) -> Metrics:
    """compute_metrics, metrics.cpp:16-35 (host arithmetic, same expressions)."""
    m = Metrics()
    tp, tn, fp, fn = float(c.tp), float(c.tn), float(c.fp), float(c.fn)
    if c.tp + c.fp == 0:
        m.precision_defined = False
    else:
        m.precision = tp / (tp + fp)
    if c.tp + c.fn == 0:
        m.recall_defined = False
    else:
        m.recall = tp / (tp + fn)
    total = tp + tn + fp + fn
    m.accuracy = 0.0 if total == 0.0 else (tp + tn) / total
    return m


def porosity(img: BinaryImage) -> float:
    """porosity, metrics.cpp:37-42: fraction of pixels equal to 1."""
    px = np.asarray(img.pixels, np.uint8)
    if px.size == 0:
        return 0.0
    return float(int(px.astype(np.uint64).sum())) / float(px.size)


# ---- label maps and RLM1 I/O (proj/include/dpmrf/graph/label_map.hpp) ------------------
@dataclass
class LabelMap:
    """LabelMap, label_map.hpp:12-17: row-major region ids; num_regions is set
    by validation."""
    width: int
    height: int
    region: np.ndarray
    num_regions: int = 0


def validate_label_map(m: LabelMap, backend: Backend = Backend.cuda()) -> LabelMap:
    """validate_label_map (label_map.cpp:38-78), on the device; fills num_regions."""
    if np.asarray(m.region).size != m.width * m.height:  # (:40, before any device work)
        raise InputError("label map: size does not match dimensions")
    m.num_regions = context_for(backend).validate_label_map(m.width, m.height, m.region)
    return m


def read_rlm(path: str, backend: Backend = Backend.cuda()) -> LabelMap:
    """read_rlm, label_map.cpp:114-133: 'RLM1', u32le width, height, then
    width*height u32le ids; InputError on a bad magic, zero dimension, an image
    over 2^31 pixels or truncation; the map is validated (on the device)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise InputError("cannot open " + path) from None
    if len(data) < 4 or data[:4] != b"RLM1":
        raise InputError(path + ": not an RLM1 file")
    if len(data) < 12:
        raise InputError(path + ": truncated")
    w, h = (int(x) for x in np.frombuffer(data, "<u4", 2, 4))
    if w == 0 or h == 0:
        raise InputError(path + ": zero dimension")
    n = w * h
    if n > (1 << 31):
        raise InputError(path + ": image too large")
    if len(data) < 12 + 4 * n:
        raise InputError(path + ": truncated")
    region = np.frombuffer(data, "<u4", n, 12).astype(np.uint32)
    return validate_label_map(LabelMap(w, h, region), backend)


def write_rlm(m: LabelMap, path: str) -> None:
    """write_rlm, label_map.cpp:135-145."""
    region = np.asarray(m.region)
    if region.size != m.width * m.height:
        raise InputError("rlm write: region buffer does not match dimensions")
    try:
        with open(path, "wb") as f:
            f.write(b"RLM1")
            f.write(np.array([m.width, m.height], "<u4").tobytes())
            f.write(region.astype("<u4").tobytes())
    except OSError:
        raise InputError("rlm write failed: " + path) from None
