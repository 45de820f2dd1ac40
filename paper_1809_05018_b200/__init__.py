"""B200-native DPP-PMRF optimization hot path (arXiv 1809.05018).

The product is the C ABI in include/dpmrf_cuda.h, implemented by hand-written
sm_100a kernels in csrc/ (libdpmrf_cuda.so).  This package is the host-side
mirror of the reference's engine interface (engine.py) plus synthetic input
construction (inputs.py).
"""
from .engine import (Backend, CliqueSet, Context, CudaError, EmIterationLog, InputError,  # noqa
                     LabelParams, MapIterationLog, MinLabelEnergies, NeighborhoodSet,
                     OptimizeResult, OptimizerConfig, RegionGraph, ReplicatedIndex,
                     TRACE_EM, TRACE_FULL, TRACE_NONE, build_neighborhoods, check_convergence,
                     compute_energies, discord_counts, init_random, min_label_energies,
                     neighborhood_energy_sums, optimize, replicate_by_label, slot_hood_map,
                     update_labels, update_parameters, PartitionGroup, nccl_unique_id)

__all__ = [n for n in dir() if not n.startswith("_")]
