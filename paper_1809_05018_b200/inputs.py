"""Synthetic inputs of the named benchmark shapes (host side).

phantom -> corrupt -> oversegment (grid or brick) -> region graph -> maximal
cliques, with the reference's semantics (proj/src/eval/phantom.cpp,
proj/src/graph/{label_map,region_graph,cliques}.cpp), built by
libdpmrf_inputs.so.  The neighborhoods are then built ON THE DEVICE by
``engine.build_neighborhoods`` (or the C ABI's dpmrf_build_neighborhoods).
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import CliqueSet, InputError, RegionGraph


@dataclass
class PhantomSpec:
    """PhantomSpec, proj/include/dpmrf/eval/phantom.hpp:9-17."""

    width: int = 128
    height: int = 128
    pore_fraction: float = 0.25
    sp_rate: float = 0.0
    gauss_sigma: float = 0.0
    ringing: bool = False
    seed: int = 0


@dataclass
class Slice:
    image: np.ndarray     # u8, row-major
    truth: np.ndarray     # u8 {0,1}
    region: np.ndarray    # u32 region id per pixel
    graph: RegionGraph
    cliques: CliqueSet


def gen_phantom(spec: PhantomSpec):
    L = N.inputs()
    n = spec.width * spec.height
    truth, clean = np.zeros(n, np.uint8), np.zeros(n, np.uint8)
    if L.dpmrf_in_phantom(spec.width, spec.height, spec.pore_fraction, spec.seed, N.ptr(truth),
                          N.ptr(clean)):
        raise InputError("phantom: invalid spec")
    return truth, clean


def corrupt(clean: np.ndarray, spec: PhantomSpec) -> np.ndarray:
    out = np.zeros_like(clean)
    if N.inputs().dpmrf_in_corrupt(N.ptr(clean), spec.width, spec.height, spec.sp_rate,
                                   spec.gauss_sigma, int(spec.ringing), spec.seed, N.ptr(out)):
        raise InputError("phantom: invalid spec")
    return out


def oversegment(width, height, block, brick=False):
    region = np.zeros(width * height, np.uint32)
    fn = N.inputs().dpmrf_in_brick_oversegment if brick else N.inputs().dpmrf_in_grid_oversegment
    R = fn(width, height, block, N.ptr(region))
    if R == 0:
        raise InputError("oversegment: invalid size")
    return region, int(R)


def region_graph(width, height, pixels, region, R) -> RegionGraph:
    L = N.inputs()
    A = ct.c_uint64(0)
    h = L.dpmrf_in_region_graph(width, height, N.ptr(pixels), N.ptr(region), R, ct.byref(A))
    if not h:
        raise InputError("region graph: invalid label map")
    try:
        off = np.zeros(R + 1, np.uint32)
        nbr = np.zeros(A.value, np.uint32)
        mean = np.zeros(R)
        size = np.zeros(R, np.uint32)
        L.dpmrf_in_graph_arrays(h, N.ptr(off), N.ptr(nbr), N.ptr(mean), N.ptr(size))
    finally:
        L.dpmrf_in_graph_free(h)
    return RegionGraph(off, nbr, mean, size)


def maximal_cliques(graph: RegionGraph) -> CliqueSet:
    L = N.inputs()
    C, CS = ct.c_uint64(0), ct.c_uint64(0)
    off_in = np.ascontiguousarray(graph.offsets, np.uint32)
    nbr_in = np.ascontiguousarray(graph.neighbors, np.uint32)
    h = L.dpmrf_in_maximal_cliques(graph.num_vertices, N.ptr(off_in), N.ptr(nbr_in) or 0,
                                   ct.byref(C), ct.byref(CS))
    try:
        off = np.zeros(C.value + 1, np.uint32)
        mem = np.zeros(CS.value, np.uint32)
        L.dpmrf_in_clique_arrays(h, N.ptr(off), N.ptr(mem))
    finally:
        L.dpmrf_in_cliques_free(h)
    return CliqueSet(off, mem)


def synthetic_slice(size=2560, block=8, brick=False, seed=42, pore=0.25, sp=0.05, gauss=100.0,
                    ringing=True, height=None) -> Slice:
    """The BASELINE.json synthetic slice: phantom{pore .25, s&p .05, gauss 100,
    ringing, seed} -> grid (or brick) oversegmentation -> graph -> cliques."""
    spec = PhantomSpec(size, height or size, pore, sp, gauss, ringing, seed)
    truth, clean = gen_phantom(spec)
    image = corrupt(clean, spec)
    region, R = oversegment(spec.width, spec.height, block, brick)
    g = region_graph(spec.width, spec.height, image, region, R)
    return Slice(image, truth, region, g, maximal_cliques(g))
