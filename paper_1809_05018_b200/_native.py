"""ctypes bindings of the in-tree native libraries.

``libdpmrf_cuda.so``   -- the C ABI of include/dpmrf_cuda.h (sm_100a kernels)
``libdpmrf_inputs.so`` -- host-side synthetic input construction

There is no fallback: if the CUDA library is missing or fails to load, every
entry point raises.  Build with ``python -c "import __graft_entry__ as g; g.build()"``
or ``make -C paper_1809_05018_b200/csrc``.
"""
from __future__ import annotations

import ctypes as ct
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# DPMRF_CUDA_LIB overrides the path (A/B builds of the same library, tools/ab.py)
CUDA_LIB = os.environ.get("DPMRF_CUDA_LIB") or os.path.join(HERE, "libdpmrf_cuda.so")
INPUTS_LIB = os.path.join(HERE, "libdpmrf_inputs.so")

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
VP = ct.c_void_p
U32, U64, I32, F64, INT = ct.c_uint32, ct.c_uint64, ct.c_int32, ct.c_double, ct.c_int
ST = ct.c_int  # dpmrf_status


class CConfig(ct.Structure):
    """dpmrf_optimizer_config == OptimizerConfig (model.hpp:19-27)."""

    _fields_ = [("num_labels", U32), ("em_max_iters", I32), ("map_max_iters", I32),
                ("convergence_window", I32), ("convergence_tol", F64), ("beta", F64),
                ("rng_seed", U64)]


class CRunOptions(ct.Structure):
    _fields_ = [("flags", U32), ("trace_level", I32)]


class CRunStats(ct.Structure):
    _fields_ = [("optimize_ms", F64), ("vertex_kernel_ms", F64), ("hood_kernel_ms", F64),
                ("mstep_ms", F64), ("vertex_launches", U64), ("hood_launches", U64),
                ("kernel_launches", U64), ("em_iters", I32), ("map_iters_total", I32),
                ("series", U64), ("map_loop_ms", F64), ("map_loop_launches", U64),
                ("active_set", I32), ("graphs", I32), ("device_loop", I32),
                ("device_log_fallbacks", U32), ("packed_layout", U32), ("reserved0", U32)]


class CPhantomSpec(ct.Structure):
    """dpmrf_phantom_spec == PhantomSpec (phantom.hpp:9-17)."""

    _fields_ = [("width", U32), ("height", U32), ("pore_fraction", F64), ("sp_rate", F64),
                ("gauss_sigma", F64), ("ringing", I32), ("seed", U64)]


class CGroupInfo(ct.Structure):
    """dpmrf_group_info."""

    _fields_ = [("world", I32), ("rank", I32), ("vertex_begin", U32), ("vertex_end", U32),
                ("series_begin", U64), ("series_end", U64), ("halo_bytes_per_map", U64),
                ("gather_bytes_per_em", U64)]


# (name, restype, argtypes) of every C ABI entry point (include/dpmrf_cuda.h)
CUDA_API = [
    ("dpmrf_context_create", ST, [INT, ct.POINTER(VP)]),
    ("dpmrf_context_destroy", None, [VP]),
    ("dpmrf_last_error", ct.c_char_p, []),
    ("dpmrf_abi_version", INT, []),
    ("dpmrf_set_graph", ST, [VP, U32, VP, VP, VP]),
    ("dpmrf_set_hoods", ST, [VP, U64, VP, VP]),
    ("dpmrf_build_neighborhoods", ST, [VP, U64, VP, VP, U32, ct.POINTER(U64)]),
    ("dpmrf_get_hoods", ST, [VP, ct.POINTER(U64), ct.POINTER(U64), VP, VP, VP]),
    ("dpmrf_make_phantom", ST, [VP, ct.POINTER(CPhantomSpec), VP, VP, ct.POINTER(U32)]),
    ("dpmrf_oversegment", ST, [VP, U32, I32, ct.POINTER(U32), VP]),
    ("dpmrf_confusion", ST, [VP, U64, VP, VP, VP]),
    ("dpmrf_validate_label_map", ST, [VP, U32, U32, VP, ct.POINTER(U32)]),
    ("dpmrf_segment_mask", ST, [VP, U32, VP, VP, VP, VP]),
    ("dpmrf_build_region_graph_resident", ST, [VP, ct.POINTER(U64)]),
    ("dpmrf_build_region_graph", ST, [VP, U32, U32, VP, VP, U32, ct.POINTER(U64)]),
    ("dpmrf_build_region_graph_device", ST, [VP, U32, U32, VP, VP, U32, ct.POINTER(U64)]),
    ("dpmrf_get_graph", ST, [VP, ct.POINTER(U32), ct.POINTER(U64), VP, VP, VP, VP]),
    ("dpmrf_enumerate_maximal_cliques", ST, [VP, ct.POINTER(U64), ct.POINTER(U64)]),
    ("dpmrf_get_cliques", ST, [VP, VP, VP]),
    ("dpmrf_build_neighborhoods_resident", ST, [VP, U32, ct.POINTER(U64)]),
    ("dpmrf_optimize", ST, [VP, ct.POINTER(CConfig), ct.POINTER(CRunOptions), VP, VP, VP]),
    ("dpmrf_optimize_arrays", ST, [VP, U32, VP, VP, VP, U64, VP, VP, ct.POINTER(CConfig),
                                   ct.POINTER(CRunOptions), VP, VP, VP]),
    ("dpmrf_trace_info", ST, [VP, ct.POINTER(I32), ct.POINTER(U64)]),
    ("dpmrf_trace_em", ST, [VP, I32, ct.POINTER(I32), ct.POINTER(F64), ct.POINTER(ct.c_uint8),
                            VP, VP]),
    ("dpmrf_trace_map", ST, [VP, I32, I32, VP, VP]),
    ("dpmrf_set_trace_sink", ST, [VP, VP, VP, U64, U64]),
    ("dpmrf_get_stats", ST, [VP, ct.POINTER(CRunStats)]),
    ("dpmrf_init_random", ST, [VP, U32, U32, U64, INT, VP, VP, VP]),
    ("dpmrf_replicate_by_label", ST, [VP, U32, VP, VP, VP]),
    ("dpmrf_slot_hood_map", ST, [VP, VP]),
    ("dpmrf_discord_counts", ST, [VP, VP, U32, VP]),
    ("dpmrf_compute_energies", ST, [VP, U64, VP, VP, U32, VP, VP, VP, F64, VP]),
    ("dpmrf_min_label_energies", ST, [VP, U64, VP, VP, VP, U64, VP, VP]),
    ("dpmrf_neighborhood_energy_sums", ST, [VP, U64, VP, VP, VP, ct.POINTER(U64)]),
    ("dpmrf_check_convergence", ST, [VP, U64, U64, VP, I32, F64, VP]),
    ("dpmrf_update_labels", ST, [VP, VP, U32, VP, VP]),
    ("dpmrf_update_parameters", ST, [VP, VP, U32, VP, VP, VP, VP]),
    ("dpmrf_debug_log", ST, [VP, U64, VP, VP]),
    ("dpmrf_nccl_unique_id", ST, [VP]),
    ("dpmrf_group_create_nccl", ST, [VP, VP, INT, INT, ct.POINTER(VP)]),
    ("dpmrf_group_create_local", ST, [VP, INT, ct.POINTER(VP)]),
    ("dpmrf_group_destroy", None, [VP]),
    ("dpmrf_group_info_get", ST, [VP, VP]),
    ("dpmrf_optimize_partitioned", ST, [VP, ct.POINTER(CConfig), ct.POINTER(CRunOptions), VP, VP,
                                        VP]),
]

INPUTS_API = [
    ("dpmrf_in_phantom", INT, [U32, U32, F64, U64, VP, VP]),
    ("dpmrf_in_corrupt", INT, [VP, U32, U32, F64, F64, INT, U64, VP]),
    ("dpmrf_in_grid_oversegment", U32, [U32, U32, U32, VP]),
    ("dpmrf_in_brick_oversegment", U32, [U32, U32, U32, VP]),
    ("dpmrf_in_region_graph", VP, [U32, U32, VP, VP, U32, ct.POINTER(U64)]),
    ("dpmrf_in_graph_arrays", None, [VP, VP, VP, VP, VP]),
    ("dpmrf_in_graph_free", None, [VP]),
    ("dpmrf_in_maximal_cliques", VP, [U32, VP, VP, ct.POINTER(U64), ct.POINTER(U64)]),
    ("dpmrf_in_clique_arrays", None, [VP, VP, VP]),
    ("dpmrf_in_cliques_free", None, [VP]),
]

_cuda = None
_inputs = None


class NativeLibraryMissing(RuntimeError):
    pass


def _load(path, api):
    if not os.path.exists(path):
        raise NativeLibraryMissing(
            f"{os.path.basename(path)} is not built; run __graft_entry__.build() "
            "(the CUDA path has no fallback)")
    lib = ct.CDLL(path)
    for name, res, args in api:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def _prefer_bundled_nccl():
    """The NCCL transport dlopens libnccl.so.2 on first use.  In a Python
    process that also uses PyTorch, load the NCCL wheel torch links against
    (nvidia/nccl/lib): a libnccl.so.2 loaded first from the system path would
    be reused for torch's own dependency and lacks symbols torch needs."""
    if os.environ.get("DPMRF_NCCL_LIB"):
        return
    for base in sys.path:
        cand = os.path.join(base, "nvidia", "nccl", "lib", "libnccl.so.2")
        if base and os.path.exists(cand):
            os.environ["DPMRF_NCCL_LIB"] = cand
            return


def cuda():
    global _cuda
    if _cuda is None:
        _prefer_bundled_nccl()
        _cuda = _load(CUDA_LIB, CUDA_API)
    return _cuda


def inputs():
    global _inputs
    if _inputs is None:
        _inputs = _load(INPUTS_LIB, INPUTS_API)
    return _inputs


def ptr(a):
    """Raw pointer of a contiguous numpy array (None for empty/None)."""
    if a is None:
        return None
    return a.ctypes.data if a.size else None
