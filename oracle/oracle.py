"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

``C`` binds the C restatement (always built by ``make -C oracle``);
``Ref`` binds the reference itself (``oracle/_ref``), which exists only where
``/root/reference`` was present at build time (this container) -- the built
``.so`` also travels to the GPU box, so ``ref_available()`` is usually True
there too.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_C = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libdpmrf_ref.so")

STATUS_NAMES = {1: "InputError", 2: "invalid_argument", 3: "out_of_range", 6: "internal"}


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {STATUS_NAMES.get(code, code)}")
        self.code = code


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
VP = ct.c_void_p
U32, U64, I32, F64 = ct.c_uint32, ct.c_uint64, ct.c_int32, ct.c_double


class Config(ct.Structure):
    """OptimizerConfig, proj/include/dpmrf/mrf/model.hpp:19-27 (same defaults)."""

    _fields_ = [
        ("num_labels", U32),
        ("em_max_iters", I32),
        ("map_max_iters", I32),
        ("convergence_window", I32),
        ("convergence_tol", F64),
        ("beta", F64),
        ("rng_seed", U64),
    ]

    def __init__(self, num_labels=2, em_max_iters=20, map_max_iters=10, convergence_window=3,
                 convergence_tol=1e-4, beta=1.0, rng_seed=0):
        super().__init__(num_labels, em_max_iters, map_max_iters, convergence_window,
                         convergence_tol, beta, rng_seed)


class _Trace(ct.Structure):
    _fields_ = [
        ("em_map_iters", VP),
        ("em_total", VP),
        ("em_conv", VP),
        ("em_mu", VP),
        ("em_sigma", VP),
        ("map_energy", VP),
        ("map_conv", VP),
        ("em_iters", I32),
        ("series", U64),
    ]


@dataclass
class Graph:
    """RegionGraph, proj/include/dpmrf/graph/region_graph.hpp:14-25."""

    offsets: np.ndarray
    neighbors: np.ndarray
    region_mean: np.ndarray

    @property
    def num_vertices(self) -> int:
        return len(self.offsets) - 1


@dataclass
class Hoods:
    """NeighborhoodSet, proj/include/dpmrf/graph/neighborhoods.hpp:15-23."""

    offsets: np.ndarray
    members: np.ndarray

    @property
    def size(self) -> int:
        return len(self.offsets) - 1


@dataclass
class MapLog:
    hood_energy: np.ndarray
    converged: np.ndarray


@dataclass
class EmLog:
    map_iters: List[MapLog]
    total_energy: float
    converged: bool
    mu: np.ndarray
    sigma: np.ndarray
    num_map_iters: int = 0


@dataclass
class Result:
    labels: np.ndarray
    mu: np.ndarray
    sigma: np.ndarray
    trace: List[EmLog] = field(default_factory=list)
    seconds: float = 0.0


def _a(x, dt):
    return np.ascontiguousarray(np.asarray(x, dtype=dt))


class _Buffers:
    def __init__(self, cfg: Config, H: int, full: bool):
        M, em, mp = cfg.num_labels, max(cfg.em_max_iters, 1), cfg.map_max_iters
        self.em_map_iters = np.zeros(em, np.int32)
        self.em_total = np.zeros(em, np.float64)
        self.em_conv = np.zeros(em, np.uint8)
        self.em_mu = np.zeros(em * M, np.float64)
        self.em_sigma = np.zeros(em * M, np.float64)
        self.map_energy = np.zeros(em * mp * max(H, 1), np.float64) if full else None
        self.map_conv = np.zeros(em * mp * max(H, 1), np.uint8) if full else None
        self.t = _Trace(self.em_map_iters.ctypes.data, self.em_total.ctypes.data,
                        self.em_conv.ctypes.data, self.em_mu.ctypes.data, self.em_sigma.ctypes.data,
                        self.map_energy.ctypes.data if full else None,
                        self.map_conv.ctypes.data if full else None, 0, 0)

    def trace(self, cfg: Config, H: int) -> List[EmLog]:
        M, mp = cfg.num_labels, cfg.map_max_iters
        out = []
        series = int(self.t.series)
        for em in range(self.t.em_iters):
            n = int(self.em_map_iters[em])
            maps = []
            if self.map_energy is not None:
                for it in range(n):
                    b = (em * mp + it) * H
                    maps.append(MapLog(self.map_energy[b:b + series].copy(),
                                       self.map_conv[b:b + series].copy()))
            out.append(EmLog(maps, float(self.em_total[em]), bool(self.em_conv[em]),
                             self.em_mu[em * M:(em + 1) * M].copy(),
                             self.em_sigma[em * M:(em + 1) * M].copy(), n))
        return out


# --------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------
class _COracle:
    def __init__(self):
        if not os.path.exists(LIB_C):
            build()
        L = ct.CDLL(LIB_C)
        self.L = L
        L.orc_init_random.argtypes = [U32, U32, U64, ct.c_int, f64p, f64p, u32p]
        L.orc_fold_range_add.argtypes = [f64p, ct.c_size_t]
        L.orc_fold_range_add.restype = F64
        L.orc_fold_tree_add.argtypes = [f64p, ct.c_size_t]
        L.orc_fold_tree_add.restype = F64
        L.orc_reduce_add.argtypes = [f64p, ct.c_size_t]
        L.orc_reduce_add.restype = F64
        L.orc_slot_hood_map.argtypes = [U64, u32p, u32p]
        L.orc_replicate_by_label.argtypes = [U64, u32p, U32, u32p, u32p, u32p]
        L.orc_discord_counts.argtypes = [U32, u32p, u32p, u32p, U32, u32p]
        L.orc_label_terms.argtypes = [U32, f64p, f64p, f64p, f64p, f64p]
        L.orc_label_energy_pub.argtypes = [F64, F64, F64, F64, F64, U32]
        L.orc_label_energy_pub.restype = F64
        L.orc_compute_energies.argtypes = [U32, u32p, u32p, f64p, U64, u32p, U64, u32p, u32p, U32,
                                           f64p, f64p, u32p, F64, f64p]
        L.orc_min_label_energies.argtypes = [U64, u32p, u32p, f64p, U64, f64p, u32p]
        L.orc_neighborhood_energy_sums.argtypes = [U64, u32p, f64p, f64p, ct.POINTER(U64)]
        L.orc_check_convergence.argtypes = [U64, U64, f64p, ct.c_int, F64, u8p]
        L.orc_update_labels.argtypes = [U64, u32p, u32p, U32, u32p, u32p]
        L.orc_update_parameters.argtypes = [U32, f64p, u32p, U32, f64p, f64p, f64p, f64p]
        L.orc_build_neighborhoods.argtypes = [U32, u32p, u32p, U64, u32p, u32p, U32, VP, VP, VP,
                                              ct.POINTER(U64)]
        PU32 = ct.POINTER(ct.POINTER(ct.c_uint32))
        L.orc_region_graph.argtypes = [U32, U32, u8p, u32p, U32, u32p, PU32, ct.POINTER(U64), f64p,
                                       u32p]
        L.orc_maximal_cliques.argtypes = [U32, u32p, u32p, PU32, ct.POINTER(U64), PU32,
                                          ct.POINTER(U64)]
        L.orc_free.argtypes = [VP]
        L.orc_confusion.argtypes = [U64, u8p, u8p, ct.POINTER(U64)]
        L.orc_labels_to_mask.argtypes = [U64, u32p, u32p, f64p, u8p]
        L.orc_validate_label_map.argtypes = [U32, U32, u32p, ct.POINTER(U32),
                                             ct.POINTER(ct.c_int), ct.POINTER(U32)]
        for fn in (L.orc_optimize, L.orc_optimize_reference):
            fn.argtypes = [U32, u32p, u32p, f64p, U64, u32p, u32p, ct.POINTER(Config), ct.c_int,
                           ct.c_int, u32p, f64p, f64p, ct.POINTER(_Trace)]

    @staticmethod
    def _chk(rc, where):
        if rc:
            raise OracleError(rc, where)

    def init_random(self, M, R, seed, allow_multilabel=False):
        mu, sig, lab = np.zeros(M), np.zeros(M), np.zeros(R, np.uint32)
        self._chk(self.L.orc_init_random(M, R, seed, int(allow_multilabel), mu, sig, lab),
                  "init_random")
        return mu, sig, lab

    def fold_range(self, x):
        x = _a(x, np.float64)
        return self.L.orc_fold_range_add(x, len(x))

    def fold_tree(self, partials):
        """fold_tree<plus> (kernels.hpp:45-51) over leaf partials (len >= 1)."""
        p = _a(partials, np.float64)
        return self.L.orc_fold_tree_add(p, len(p))

    def reduce(self, x):
        x = _a(x, np.float64)
        return self.L.orc_reduce_add(x, len(x)) if len(x) else 0.0

    def slot_hood_map(self, hoods: Hoods):
        out = np.zeros(int(hoods.offsets[-1]), np.uint32)
        self.L.orc_slot_hood_map(hoods.size, _a(hoods.offsets, np.uint32), out)
        return out

    def replicate_by_label(self, hoods: Hoods, M):
        E = int(hoods.offsets[-1]) * M
        tl, oi, hid = (np.zeros(E, np.uint32) for _ in range(3))
        self.L.orc_replicate_by_label(hoods.size, _a(hoods.offsets, np.uint32), M, tl, oi, hid)
        return tl, oi, hid

    def discord_counts(self, g: Graph, labels, M):
        out = np.zeros(M * g.num_vertices, np.uint32)
        self.L.orc_discord_counts(g.num_vertices, _a(g.offsets, np.uint32),
                                  _a(g.neighbors, np.uint32), _a(labels, np.uint32), M, out)
        return out

    def label_terms(self, mu, sigma):
        mu, sigma = _a(mu, np.float64), _a(sigma, np.float64)
        M = len(mu)
        a, b, c = np.zeros(M), np.zeros(M), np.zeros(M)
        self.L.orc_label_terms(M, mu, sigma, a, b, c)
        return a, b, c

    def label_energy(self, x, mu, two_var, log_sigma, beta, discord):
        return self.L.orc_label_energy_pub(x, mu, two_var, log_sigma, beta, discord)

    def compute_energies(self, g: Graph, hoods: Hoods, rep, mu, sigma, labels, beta):
        tl, oi, _ = rep
        out = np.zeros(len(tl))
        rc = self.L.orc_compute_energies(
            g.num_vertices, _a(g.offsets, np.uint32), _a(g.neighbors, np.uint32),
            _a(g.region_mean, np.float64), len(hoods.members), _a(hoods.members, np.uint32),
            len(tl), _a(tl, np.uint32), _a(oi, np.uint32), len(mu), _a(mu, np.float64),
            _a(sigma, np.float64), _a(labels, np.uint32), beta, out)
        self._chk(rc, "compute_energies")
        return out

    def min_label_energies(self, rep, energies, num_slots):
        tl, oi = rep[0], rep[1]
        oe, ol = np.zeros(num_slots), np.zeros(num_slots, np.uint32)
        rc = self.L.orc_min_label_energies(len(tl), _a(tl, np.uint32), _a(oi, np.uint32),
                                           _a(energies, np.float64), num_slots, oe, ol)
        self._chk(rc, "min_label_energies")
        return oe, ol

    def neighborhood_energy_sums(self, slot_hood, mins):
        out = np.zeros(max(len(slot_hood), 1))
        n = U64(0)
        self.L.orc_neighborhood_energy_sums(len(slot_hood), _a(slot_hood, np.uint32),
                                            _a(mins, np.float64), out, ct.byref(n))
        return out[:n.value].copy()

    def check_convergence(self, history, window, tol):
        if len(history) == 0:
            return np.zeros(0, np.uint8)
        h = _a(np.asarray(history, dtype=np.float64).reshape(len(history), -1), np.float64)
        out = np.zeros(h.shape[1], np.uint8)
        self.L.orc_check_convergence(h.shape[0], h.shape[1], h.ravel(), window, tol, out)
        return out

    def update_labels(self, hoods: Hoods, argmin, old_labels):
        old = _a(old_labels, np.uint32)
        out = np.zeros(len(old), np.uint32)
        rc = self.L.orc_update_labels(len(hoods.members), _a(hoods.members, np.uint32),
                                      _a(argmin, np.uint32), len(old), old, out)
        self._chk(rc, "update_labels")
        return out

    def update_parameters(self, region_mean, labels, prev_mu, prev_sigma):
        M = len(prev_mu)
        mu, sig = np.zeros(M), np.zeros(M)
        rc = self.L.orc_update_parameters(len(region_mean), _a(region_mean, np.float64),
                                          _a(labels, np.uint32), M, _a(prev_mu, np.float64),
                                          _a(prev_sigma, np.float64), mu, sig)
        self._chk(rc, "update_parameters")
        return mu, sig

    def build_neighborhoods(self, g: Graph, c_off, c_mem, k=1):
        c_off, c_mem = _a(c_off, np.uint32), _a(c_mem, np.uint32)
        C = len(c_off) - 1
        n = U64(0)
        args = (g.num_vertices, _a(g.offsets, np.uint32), _a(g.neighbors, np.uint32), C, c_off,
                c_mem, k)
        self._chk(self.L.orc_build_neighborhoods(*args, None, None, None, ct.byref(n)),
                  "build_neighborhoods")
        off = np.zeros(C + 1, np.uint32)
        mem = np.zeros(max(n.value, 1), np.uint32)
        src = np.zeros(max(C, 1), np.uint32)
        self._chk(self.L.orc_build_neighborhoods(*args, off.ctypes.data, mem.ctypes.data,
                                                 src.ctypes.data, ct.byref(n)),
                  "build_neighborhoods")
        return Hoods(off, mem[:n.value].copy()), src[:C].copy()

    def _run(self, fn, g: Graph, hoods: Hoods, cfg: Config, fixed_work, allow_multilabel, full):
        R, M = g.num_vertices, cfg.num_labels
        lab, mu, sig = np.zeros(R, np.uint32), np.zeros(M), np.zeros(M)
        buf = _Buffers(cfg, hoods.size, full)
        rc = fn(R, _a(g.offsets, np.uint32), _a(g.neighbors, np.uint32),
                _a(g.region_mean, np.float64), hoods.size, _a(hoods.offsets, np.uint32),
                _a(hoods.members, np.uint32), ct.byref(cfg), int(fixed_work),
                int(allow_multilabel), lab, mu, sig, ct.byref(buf.t))
        self._chk(rc, fn.__name__)
        return Result(lab, mu, sig, buf.trace(cfg, hoods.size))

    def _take(self, p, n):
        out = np.ctypeslib.as_array(p, shape=(max(n, 1),))[:n].copy() if n else \
            np.zeros(0, np.uint32)
        self.L.orc_free(ct.cast(p, VP))
        return out

    def region_graph(self, width, height, pixels, region, R):
        """build_region_graph (region_graph.cpp:10-73) -> (Graph, region_size)."""
        off = np.zeros(R + 1, np.uint32)
        mean, size = np.zeros(max(R, 1)), np.zeros(max(R, 1), np.uint32)
        nbr_p, A = ct.POINTER(ct.c_uint32)(), U64(0)
        self._chk(self.L.orc_region_graph(width, height, _a(pixels, np.uint8), _a(region, np.uint32),
                                          R, off, ct.byref(nbr_p), ct.byref(A), mean, size),
                  "region_graph")
        return Graph(off, self._take(nbr_p, A.value), mean[:R].copy()), size[:R].copy()

    def maximal_cliques(self, g: Graph):
        """enumerate_maximal_cliques (cliques.cpp:53-106) -> (offsets, members)."""
        po, pm = ct.POINTER(ct.c_uint32)(), ct.POINTER(ct.c_uint32)()
        C, CS = U64(0), U64(0)
        nbr = _a(g.neighbors, np.uint32)
        if len(nbr) == 0:
            nbr = np.zeros(1, np.uint32)
        self._chk(self.L.orc_maximal_cliques(g.num_vertices, _a(g.offsets, np.uint32), nbr,
                                             ct.byref(po), ct.byref(C), ct.byref(pm),
                                             ct.byref(CS)), "maximal_cliques")
        off = self._take(po, C.value + 1)
        return off, self._take(pm, CS.value)

    def confusion(self, pred, truth):
        """confusion_u8 (scalar_kernels.cpp:48-63) -> (tp, tn, fp, fn)."""
        a, b = _a(pred, np.uint8), _a(truth, np.uint8)
        c = (U64 * 4)()
        self.L.orc_confusion(a.size, a, b, c)
        return tuple(int(x) for x in c)

    def validate_label_map(self, w, h, region):
        """label_map.cpp:38-78 -> num_regions, or the reference's InputError
        message (as a string) when the map is invalid."""
        reg = _a(region, np.uint32) if len(region) else np.zeros(1, np.uint32)
        num, kind, det = U32(0), ct.c_int(0), U32(0)
        rc = self.L.orc_validate_label_map(w, h, reg, ct.byref(num), ct.byref(kind),
                                           ct.byref(det))
        if rc == 0:
            return num.value
        if kind.value == 1:
            return f"label map: region id {det.value} unused"
        if kind.value == 2:
            return f"label map: region {det.value} is not 4-connected"
        if kind.value == 3:
            return "label map: empty"
        raise OracleError(rc, "validate_label_map")

    def labels_to_mask(self, region, labels, mu):
        """main.cpp:157-165 -> u8 mask."""
        reg = _a(region, np.uint32)
        out = np.zeros(reg.size, np.uint8)
        self.L.orc_labels_to_mask(reg.size, reg, _a(labels, np.uint32), _a(mu, np.float64), out)
        return out

    def optimize(self, g, hoods, cfg, fixed_work=False, allow_multilabel=False, full_trace=True):
        return self._run(self.L.orc_optimize, g, hoods, cfg, fixed_work, allow_multilabel,
                         full_trace)

    def optimize_reference(self, g, hoods, cfg, fixed_work=False, allow_multilabel=False):
        return self._run(self.L.orc_optimize_reference, g, hoods, cfg, fixed_work,
                         allow_multilabel, False)


# --------------------------------------------------------------------------
# The reference itself
# --------------------------------------------------------------------------
def ref_available() -> bool:
    return os.path.exists(LIB_REF)


class Pipe:
    """Structures built by the reference (graph, cliques, hoods, image)."""

    def __init__(self, ref: "_Ref", handle):
        self.ref, self.h = ref, handle
        sz = np.zeros(8, np.uint64)
        ref.L.ref_pipe_sizes(handle, sz)
        self.R, self.A, self.C, self.CS, self.H, self.S, self.W, self.HP = (int(x) for x in sz)

    def __del__(self):
        try:
            self.ref.L.ref_pipe_free(self.h)
        except Exception:
            pass

    def graph(self) -> Graph:
        off = np.zeros(self.R + 1, np.uint32)
        nbr = np.zeros(max(self.A, 1), np.uint32)
        mean = np.zeros(max(self.R, 1))
        size = np.zeros(max(self.R, 1), np.uint32)
        self.ref.L.ref_pipe_graph(self.h, off, nbr, mean, size)
        return Graph(off, nbr[:self.A].copy(), mean[:self.R].copy())

    def cliques(self):
        off = np.zeros(self.C + 1, np.uint32)
        mem = np.zeros(max(self.CS, 1), np.uint32)
        self.ref.L.ref_pipe_cliques(self.h, off, mem)
        return off, mem[:self.CS].copy()

    def hoods(self) -> Hoods:
        off = np.zeros(self.H + 1, np.uint32)
        mem = np.zeros(max(self.S, 1), np.uint32)
        src = np.zeros(max(self.H, 1), np.uint32)
        self.ref.L.ref_pipe_hoods(self.h, off, mem, src)
        return Hoods(off, mem[:self.S].copy())

    def image(self):
        n = self.W * self.HP
        px, tr, reg = np.zeros(n, np.uint8), np.zeros(n, np.uint8), np.zeros(n, np.uint32)
        self.ref.L.ref_pipe_image(self.h, px, tr, reg)
        return px, tr, reg

    def times(self):
        t = np.zeros(3)
        self.ref.L.ref_pipe_times(self.h, t)
        return t

    def _run(self, fn, cfg, extra, full):
        M = cfg.num_labels
        lab, mu, sig = np.zeros(self.R, np.uint32), np.zeros(M), np.zeros(M)
        buf = _Buffers(cfg, self.H, full)
        secs = F64(0)
        rc = fn(self.h, ct.byref(cfg), *extra, lab, mu, sig, ct.byref(buf.t), ct.byref(secs))
        if rc:
            raise OracleError(rc, fn.__name__)
        return Result(lab, mu, sig, buf.trace(cfg, self.H), secs.value)

    def optimize(self, cfg, threads=1, mode=0, fixed_work=False, full_trace=True):
        """mode 0: dpmrf::optimize itself; mode 1: public-step recomposition."""
        return self._run(self.ref.L.ref_optimize, cfg, (threads, mode, int(fixed_work)),
                         full_trace)

    def sweep(self, cfg, mode=0, fixed_work=False):
        """mode 0: dpmrf::optimize_reference itself; mode 1: its restated body."""
        return self._run(self.ref.L.ref_sweep, cfg, (mode, int(fixed_work)), False)

    def discord_counts(self, labels, M):
        out = np.zeros(M * self.R, np.uint32)
        rc = self.ref.L.ref_discord_counts(self.h, _a(labels, np.uint32), M, out)
        if rc:
            raise OracleError(rc, "discord_counts")
        return out

    def compute_energies(self, rep, mu, sigma, labels, beta):
        tl, oi, hid = (_a(x, np.uint32) for x in rep)
        out = np.zeros(len(tl))
        rc = self.ref.L.ref_compute_energies(self.h, len(tl), tl, oi, hid, len(mu),
                                             _a(mu, np.float64), _a(sigma, np.float64),
                                             _a(labels, np.uint32), beta, out)
        if rc:
            raise OracleError(rc, "compute_energies")
        return out


class _Ref:
    def __init__(self):
        if not ref_available():
            raise OracleError(6, "oracle/_ref/libdpmrf_ref.so not built")
        L = ct.CDLL(LIB_REF)
        self.L = L
        ip = ct.POINTER(ct.c_int)
        L.ref_pipe_phantom.argtypes = [U32, U32, F64, F64, F64, ct.c_int, U64, U32, ct.c_int,
                                       ct.c_int, ip]
        L.ref_pipe_phantom.restype = VP
        L.ref_pipe_arrays.argtypes = [U32, u32p, u32p, f64p, U64, VP, VP, U64, VP, VP, ip]
        L.ref_pipe_arrays.restype = VP
        L.ref_pipe_labelmap.argtypes = [U32, U32, u8p, u32p, U32, ct.c_int, ip]
        L.ref_pipe_labelmap.restype = VP
        L.ref_pipe_free.argtypes = [VP]
        L.ref_pipe_sizes.argtypes = [VP, np.ctypeslib.ndpointer(np.uint64)]
        L.ref_pipe_times.argtypes = [VP, f64p]
        L.ref_pipe_graph.argtypes = [VP, u32p, u32p, f64p, u32p]
        L.ref_pipe_cliques.argtypes = [VP, u32p, u32p]
        L.ref_pipe_hoods.argtypes = [VP, u32p, u32p, u32p]
        L.ref_pipe_image.argtypes = [VP, u8p, u8p, u32p]
        L.ref_optimize.argtypes = [VP, ct.POINTER(Config), ct.c_int, ct.c_int, ct.c_int, u32p,
                                   f64p, f64p, ct.POINTER(_Trace), ct.POINTER(F64)]
        L.ref_sweep.argtypes = [VP, ct.POINTER(Config), ct.c_int, ct.c_int, u32p, f64p, f64p,
                                ct.POINTER(_Trace), ct.POINTER(F64)]
        L.ref_init_random.argtypes = [U32, U32, U64, f64p, f64p, u32p]
        L.ref_replicate_by_label.argtypes = [U64, u32p, u32p, U32, u32p, u32p, u32p]
        L.ref_discord_counts.argtypes = [VP, u32p, U32, u32p]
        L.ref_compute_energies.argtypes = [VP, U64, u32p, u32p, u32p, U32, f64p, f64p, u32p, F64,
                                           f64p]
        L.ref_min_label_energies.argtypes = [U64, u32p, u32p, f64p, U64, f64p, u32p]
        L.ref_neighborhood_energy_sums.argtypes = [U64, u32p, f64p, f64p, ct.POINTER(U64)]
        L.ref_check_convergence.argtypes = [U64, U64, f64p, ct.c_int, F64, u8p, ct.POINTER(U64)]
        L.ref_update_labels.argtypes = [U64, u32p, u32p, u32p, U32, u32p, u32p]
        L.ref_update_parameters.argtypes = [U32, f64p, u32p, U32, f64p, f64p, f64p, f64p]
        L.ref_reduce_add.argtypes = [U64, f64p]
        L.ref_reduce_add.restype = F64
        L.ref_hw_threads.restype = U32
        L.ref_confusion.argtypes = [U32, U32, u8p, U32, U32, u8p, ct.POINTER(U64)]
        L.ref_compute_metrics.argtypes = [ct.POINTER(U64), ct.POINTER(F64), ct.POINTER(ct.c_int)]
        L.ref_validate_label_map.argtypes = [U32, U32, u32p, U64, ct.POINTER(U32), ct.c_char_p,
                                             U64]
        L.ref_porosity.argtypes = [U32, U32, u8p]
        L.ref_porosity.restype = F64

    def phantom(self, size=256, block=8, pore=0.25, sp=0.05, gauss=100.0, ringing=True, seed=42,
                brick=False, threads=1, height=None) -> Pipe:
        st = ct.c_int(0)
        h = self.L.ref_pipe_phantom(size, height or size, pore, sp, gauss, int(ringing), seed,
                                    block, int(brick), threads, ct.byref(st))
        if st.value:
            raise OracleError(st.value, "ref_pipe_phantom")
        return Pipe(self, h)

    def arrays(self, g: Graph, cliques=None, hoods: Optional[Hoods] = None) -> Pipe:
        st = ct.c_int(0)
        c_off = c_mem = h_off = h_mem = None
        C = H = 0
        keep = []
        if cliques is not None:
            c_off, c_mem = _a(cliques[0], np.uint32), _a(cliques[1], np.uint32)
            keep += [c_off, c_mem]
            C = len(c_off) - 1
        if hoods is not None:
            h_off, h_mem = _a(hoods.offsets, np.uint32), _a(hoods.members, np.uint32)
            if len(h_mem) == 0:
                h_mem = np.zeros(1, np.uint32)
            keep += [h_off, h_mem]
            H = len(h_off) - 1
        nbr = _a(g.neighbors, np.uint32)
        if len(nbr) == 0:
            nbr = np.zeros(1, np.uint32)
        h = self.L.ref_pipe_arrays(
            g.num_vertices, _a(g.offsets, np.uint32), nbr, _a(g.region_mean, np.float64), C,
            c_off.ctypes.data if c_off is not None else None,
            c_mem.ctypes.data if c_mem is not None else None, H,
            h_off.ctypes.data if h_off is not None else None,
            h_mem.ctypes.data if h_mem is not None else None, ct.byref(st))
        if st.value:
            raise OracleError(st.value, "ref_pipe_arrays")
        return Pipe(self, h)

    def labelmap(self, width, height, pixels, region, num_regions, threads=1) -> Pipe:
        """Graph, cliques and hoods of the caller's image + label map, by the reference."""
        st = ct.c_int(0)
        h = self.L.ref_pipe_labelmap(width, height, _a(pixels, np.uint8), _a(region, np.uint32),
                                     num_regions, threads, ct.byref(st))
        if st.value:
            raise OracleError(st.value, "ref_pipe_labelmap")
        return Pipe(self, h)

    def hw_threads(self) -> int:
        return int(self.L.ref_hw_threads())

    def confusion(self, w1, h1, pred, w2, h2, truth):
        """dpmrf::confusion on two BinaryImages -> (tp, tn, fp, fn); OracleError on
        the reference's InputError."""
        c = (U64 * 4)()
        a = _a(pred, np.uint8) if len(pred) else np.zeros(1, np.uint8)
        b = _a(truth, np.uint8) if len(truth) else np.zeros(1, np.uint8)
        rc = self.L.ref_confusion(w1, h1, a, w2, h2, b, c)
        if rc:
            raise OracleError(rc, "ref_confusion")
        return tuple(int(x) for x in c)

    def compute_metrics(self, counts):
        """dpmrf::compute_metrics -> (precision, recall, accuracy, p_def, r_def)."""
        c = (U64 * 4)(*counts)
        m = (F64 * 3)()
        d = (ct.c_int * 2)()
        self.L.ref_compute_metrics(c, m, d)
        return m[0], m[1], m[2], bool(d[0]), bool(d[1])

    def validate_label_map(self, w, h, region):
        """dpmrf::validate_label_map -> num_regions, or its what() string."""
        reg = _a(region, np.uint32) if len(region) else np.zeros(1, np.uint32)
        num, msg = U32(0), ct.create_string_buffer(256)
        rc = self.L.ref_validate_label_map(w, h, reg, len(region), ct.byref(num), msg, 256)
        return num.value if rc == 0 else msg.value.decode()

    def porosity(self, w, h, pixels):
        a = _a(pixels, np.uint8) if len(pixels) else np.zeros(1, np.uint8)
        return float(self.L.ref_porosity(w, h, a))


_C = None
_R = None


def C() -> _COracle:
    global _C
    if _C is None:
        _C = _COracle()
    return _C


def Ref() -> _Ref:
    global _R
    if _R is None:
        _R = _Ref()
    return _R


def graph_from_edges(n, edges, means=None) -> Graph:
    """make_graph of proj/tests/mrf_engine_test.cpp:20-38 (sorted, symmetric)."""
    adj = [set() for _ in range(n)]
    for a, b in edges:
        adj[a].add(b)
        adj[b].add(a)
    off, nbr = [0], []
    for v in range(n):
        nbr.extend(sorted(adj[v]))
        off.append(len(nbr))
    mean = np.full(n, 128.0) if means is None else np.asarray(means, np.float64)
    return Graph(np.asarray(off, np.uint32), np.asarray(nbr, np.uint32), mean)


def random_graph(rng: np.random.Generator, n, p, means=True) -> Graph:
    edges = [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < p]
    m = rng.uniform(0.0, 255.0, n) if means else None
    return graph_from_edges(n, edges, m)
