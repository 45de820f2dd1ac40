/*
 * dpmrf_cuda.h -- C ABI of the B200-native DPP-PMRF optimization hot path.
 *
 * The drop-in boundary for the reference's engine layer
 * (/root/reference/proj/include/dpmrf/mrf/engine.hpp:15-116 and
 *  graph/neighborhoods.hpp:28-29).  Every entry point below cites the
 * reference declaration it replaces.  Plain pointers and sizes only; no
 * exception crosses the ABI -- each call returns a dpmrf_status and leaves a
 * message for dpmrf_last_error().  The C++ drop-in (include/dpmrf_b200/
 * engine.hpp) rethrows the matching reference exception type.
 *
 * Ownership: all input pointers are caller-owned HOST memory, read during
 * the call only; all outputs are caller-allocated HOST buffers, written
 * before the call returns ("internally parallel, externally synchronous",
 * SPEC.md:126-127).  The region graph and neighborhoods are uploaded once
 * into the context and stay resident in HBM across calls.
 *
 * Threading: a context is not re-entrant (the reference thread pool
 * serializes submissions, proj/src/dpp/backend.cpp:45); use one context per
 * host thread.  Calls block until their outputs are on the host.
 */
#ifndef DPMRF_CUDA_H
#define DPMRF_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPMRF_ABI_VERSION 1

/* Error convention of the reference. */
typedef enum dpmrf_status {
  DPMRF_OK = 0,
  DPMRF_INPUT_ERROR = 1,      /* dpmrf::InputError          proj/include/dpmrf/error.hpp:11 */
  DPMRF_INVALID_ARGUMENT = 2, /* std::invalid_argument      e.g. proj/src/mrf/engine.cpp:175-176 */
  DPMRF_OUT_OF_RANGE = 3,     /* std::out_of_range          proj/include/dpmrf/dpp/kernels.hpp:313,337 */
  DPMRF_CUDA_ERROR = 4,       /* device failure (no reference counterpart) */
  DPMRF_NCCL_ERROR = 5,       /* collective failure (multi-GPU paths) */
  DPMRF_INTERNAL_ERROR = 6    /* anything else (the CLI's exit 1, proj/tools/main.cpp:248-250) */
} dpmrf_status;

typedef struct dpmrf_context dpmrf_context;

/* OptimizerConfig, proj/include/dpmrf/mrf/model.hpp:19-27 (same field order
 * and meaning; defaults 2, 20, 10, 3, 1e-4, 1.0, 0). */
typedef struct dpmrf_optimizer_config {
  uint32_t num_labels;
  int32_t em_max_iters;
  int32_t map_max_iters;
  int32_t convergence_window;
  double convergence_tol;
  double beta;
  uint64_t rng_seed;
} dpmrf_optimizer_config;

/* Run options (no reference counterpart; all-zero = reference semantics). */
enum {
  DPMRF_TRACE_NONE = 0, /* labels + params only */
  DPMRF_TRACE_EM = 1,   /* + per-EM total energy, flag, params, MAP count */
  DPMRF_TRACE_FULL = 2  /* + every MAP iteration's hood energies and flags
                           (OptimizeResult.trace, engine.hpp:82-99) */
};
enum {
  DPMRF_RUN_FIXED_WORK = 1u,    /* drop the early exits (optimize.cpp:59,:71): fixed EM x MAP work */
  DPMRF_RUN_MULTILABEL = 2u,    /* allow num_labels in [1,255] (extension; reference: 2 only) */
  DPMRF_RUN_KERNEL_TIMING = 4u, /* CUDA events around the MAP kernels (dpmrf_get_stats) */
  DPMRF_RUN_NO_GRAPH = 16u,     /* launch each EM iteration directly instead of a CUDA graph */
  /* (8u, 32u, 64u: reserved -- measured-and-rejected variants) */
  DPMRF_RUN_CSR = 256u,         /* read the u32 CSR in the MAP kernels instead of the packed
                                   int16/u16 delta layouts built at preparation */
  DPMRF_RUN_UNFUSED = 512u,     /* separate vertex and hood kernels per MAP iteration; default
                                   (packed layouts): map_max + 1 launches per EM iteration, each
                                   running the hood pass of t-1 with the vertex pass of t */
  DPMRF_RUN_HOST_LOG = 128u,    /* host round trip per EM iteration (log(sigma) on the host);
                                   default: EM iterations run back to back on the device with a
                                   correctly rounded device log, verified against the host libm
                                   afterwards (rerun with host logs on any difference) */
  DPMRF_RUN_ACTIVE_SET = 1024u  /* extension, opt-in: from the third MAP iteration of an EM on,
                                   re-evaluate only the vertices whose inputs changed (a
                                   neighbor's label) and fold only the hoods whose members'
                                   minima changed or whose window is still open; bit-identical
                                   results, but less than the reference's per-iteration work.
                                   The first EM iteration runs dense.  Grid graphs with two
                                   labels, trace levels NONE / EM, device-resident loop, one
                                   device; ignored otherwise (dpmrf_run_stats.active_set) */
};

typedef struct dpmrf_run_options {
  uint32_t flags;
  int32_t trace_level;
} dpmrf_run_options;

/* Device-side measurements of the last dpmrf_optimize call. */
typedef struct dpmrf_run_stats {
  double optimize_ms;        /* CUDA-event time of the whole optimize phase on the context stream */
  double vertex_kernel_ms;   /* sum over launches of the per-vertex energy/argmin kernel */
  double hood_kernel_ms;     /* sum over launches of the per-hood sum + convergence kernel */
  double mstep_ms;           /* M-step kernels */
  uint64_t vertex_launches;
  uint64_t hood_launches;
  uint64_t kernel_launches;  /* every kernel of this library launched by the call */
  int32_t em_iters;
  int32_t map_iters_total;   /* MAP iterations executed, summed over EM iterations */
  uint64_t series;           /* hood-energy series length (nonempty hoods) */
  double map_loop_ms;        /* fused MAP launches (events around each EM's chain of them) */
  uint64_t map_loop_launches;
  int32_t active_set;        /* 1: the active-set MAP loop ran (DPMRF_RUN_ACTIVE_SET) */
  int32_t graphs;            /* 1: EM iterations replayed from CUDA graphs */
  int32_t device_loop;       /* 1: the result came from the device-resident EM loop */
  uint32_t device_log_fallbacks; /* reruns because a device log(sigma) differed from the host's */
  uint32_t packed_layout;    /* structure layout of the MAP loop: 100 * adjacency slots + hood
                                slots (0: the CSR itself) */
  uint32_t reserved0;
} dpmrf_run_stats;

/* ---- context ------------------------------------------------------------ */
dpmrf_status dpmrf_context_create(int device, dpmrf_context** out);
void dpmrf_context_destroy(dpmrf_context* ctx);
const char* dpmrf_last_error(void); /* message of this thread's last failing call */
int dpmrf_abi_version(void);

/* ---- resident inputs ---------------------------------------------------- */
/* RegionGraph, proj/include/dpmrf/graph/region_graph.hpp:14-25: CSR with
 * num_vertices+1 offsets, offsets[R] neighbor ids, and R region means. */
dpmrf_status dpmrf_set_graph(dpmrf_context* ctx, uint32_t num_vertices, const uint32_t* offsets,
                             const uint32_t* neighbors, const double* region_mean);

/* NeighborhoodSet, proj/include/dpmrf/graph/neighborhoods.hpp:15-23:
 * num_hoods+1 offsets and offsets[num_hoods] member ids. */
dpmrf_status dpmrf_set_hoods(dpmrf_context* ctx, uint64_t num_hoods, const uint32_t* offsets,
                             const uint32_t* members);

/* build_neighborhoods, proj/include/dpmrf/graph/neighborhoods.hpp:28-29 /
 * proj/src/graph/neighborhoods.cpp:10-57: one sorted, duplicate-free
 * 1-neighborhood per maximal clique, built ON THE DEVICE from the resident
 * graph; the result becomes the context's neighborhoods.  k != 1 ->
 * DPMRF_INPUT_ERROR.  *num_slots receives the total member count. */
dpmrf_status dpmrf_build_neighborhoods(dpmrf_context* ctx, uint64_t num_cliques,
                                       const uint32_t* clique_offsets,
                                       const uint32_t* clique_members, uint32_t k,
                                       uint64_t* num_slots);

/* Copy the resident neighborhoods out (offsets: H+1, members: S,
 * source_clique: H; any pointer may be NULL). */
dpmrf_status dpmrf_get_hoods(dpmrf_context* ctx, uint64_t* num_hoods, uint64_t* num_slots,
                             uint32_t* offsets, uint32_t* members, uint32_t* source_clique);

/* ---- synthetic inputs on the device ------------ */
/* PhantomSpec, proj/include/dpmrf/eval/phantom.hpp:9-17. */
typedef struct dpmrf_phantom_spec {
  uint32_t width, height;
  double pore_fraction;  /* [0, 1) */
  double sp_rate;        /* salt-and-pepper rate, [0, 1] */
  double gauss_sigma;    /* >= 0 */
  int32_t ringing;
  uint64_t seed;
} dpmrf_phantom_spec;

/* gen_phantom + corrupt (proj/src/eval/phantom.cpp:54-150) ON THE DEVICE,
 * bit-identical to the reference: the corrupted image becomes the context's
 * resident image (input of dpmrf_build_region_graph_resident).  truth / image
 * (width*height bytes each) may be NULL, else receive copies.  *host_ties
 * (may be NULL) receives the number of pixels whose value fell within 1e-7
 * of a rounding boundary and was therefore evaluated with the host's libm.
 * An invalid spec -> DPMRF_INPUT_ERROR (validate_spec, phantom.cpp:46-52). */
dpmrf_status dpmrf_make_phantom(dpmrf_context* ctx, const dpmrf_phantom_spec* spec,
                                uint8_t* truth, uint8_t* image, uint32_t* host_ties);

/* grid_oversegment (proj/src/graph/label_map.cpp:79-94), or with brick != 0
 * the brick oversegmentation of config C (block rows of height `block`, odd
 * rows shifted by block/2, ids first-seen row-major), ON THE DEVICE for the
 * resident image's dimensions; the region map becomes resident.
 * *num_regions receives the region count; region (w*h) may be NULL. */
dpmrf_status dpmrf_oversegment(dpmrf_context* ctx, uint32_t block, int32_t brick,
                               uint32_t* num_regions, uint32_t* region);

/* validate_label_map, proj/src/graph/label_map.cpp:38-78 (called by
 * read_rlm, :131), on the device: every id in [0, max] must be used and every
 * region must be one 4-connected component.  region: width*height host ids
 * (the size check of the reference is the caller's: the buffer IS w*h).  On
 * success *num_regions = max id + 1; otherwise DPMRF_INPUT_ERROR with the
 * reference's message ("label map: empty", "label map: region id K unused" for
 * the lowest unused K, "label map: region K is not 4-connected" for the region
 * of the first pixel in scan order outside its region's first component). */
dpmrf_status dpmrf_validate_label_map(dpmrf_context* ctx, uint32_t width, uint32_t height,
                                      const uint32_t* region, uint32_t* num_regions);

/* ---- evaluation ---------------------------------
 * confusion(pred, truth), proj/include/dpmrf/eval/metrics.hpp:17-18 and
 * proj/src/eval/metrics.cpp:8-14 (simd::confusion_u8, scalar_kernels.cpp:48-63)
 * over n host pixels (nonzero = positive): counts = {tp, tn, fp, fn}.  The
 * shape check of confusion() (InputError) is the caller's (both images are n
 * pixels here). */
dpmrf_status dpmrf_confusion(dpmrf_context* ctx, uint64_t n, const uint8_t* pred,
                             const uint8_t* truth, uint64_t counts[4]);
/* The segment write-back of proj/tools/main.cpp:157-165 (== the acceptance
 * test's labels_to_mask, proj/tests/acceptance.cpp:359-370) over the resident
 * label map (dpmrf_oversegment, or the map given to dpmrf_build_region_graph): mask[p] = labels[region[p]] == pore, pore =
 * mu[0] <= mu[1] ? 0 : 1 (the darker class).  labels: num_vertices host values
 * (an optimize result, num_vertices == the map's regions); mask: width*height
 * bytes or NULL; counts: {tp, tn, fp, fn} against the resident phantom truth
 * (dpmrf_make_phantom), or NULL. */
dpmrf_status dpmrf_segment_mask(dpmrf_context* ctx, uint32_t num_vertices, const uint32_t* labels,
                                const double* mu, uint8_t* mask, uint64_t counts[4]);

/* build_region_graph from the resident image and region map. */
dpmrf_status dpmrf_build_region_graph_resident(dpmrf_context* ctx, uint64_t* num_adjacency);

/* ---- device structure builders -------------- */
/* build_region_graph, proj/include/dpmrf/graph/region_graph.hpp:31-33 /
 * proj/src/graph/region_graph.cpp:10-73, ON THE DEVICE: `pixels` is the
 * width x height u8 GrayImage (image.hpp), `region` the validated LabelMap's
 * u32 region id per pixel (label_map.hpp), num_regions its region count.
 * The graph (offsets, neighbors, region_mean, region_size) becomes the
 * context's resident graph, as after dpmrf_set_graph.  Region id >=
 * num_regions -> DPMRF_OUT_OF_RANGE; an unused id (map not validated) or
 * num_regions == 0 -> DPMRF_INPUT_ERROR (region_graph.cpp:13-15).
 * *num_adjacency (may be NULL) receives offsets[num_regions]. */
dpmrf_status dpmrf_build_region_graph(dpmrf_context* ctx, uint32_t width, uint32_t height,
                                      const uint8_t* pixels, const uint32_t* region,
                                      uint32_t num_regions, uint64_t* num_adjacency);

/* Same, with pixels / region already in device memory of the context's
 * device (no host copies; e.g. an image produced on the GPU). */
dpmrf_status dpmrf_build_region_graph_device(dpmrf_context* ctx, uint32_t width, uint32_t height,
                                             const uint8_t* pixels_dev,
                                             const uint32_t* region_dev, uint32_t num_regions,
                                             uint64_t* num_adjacency);

/* Copy the resident graph out (offsets: R+1, neighbors: A, region_mean: R,
 * region_size: R -- only for a graph built by dpmrf_build_region_graph; any
 * pointer may be NULL). */
dpmrf_status dpmrf_get_graph(dpmrf_context* ctx, uint32_t* num_vertices, uint64_t* num_adjacency,
                             uint32_t* offsets, uint32_t* neighbors, double* region_mean,
                             uint32_t* region_size);

/* enumerate_maximal_cliques, proj/include/dpmrf/graph/cliques.hpp:24-27 /
 * proj/src/graph/cliques.cpp:53-106, ON THE DEVICE over the resident graph
 * (which must satisfy RegionGraph's invariants: sorted, symmetric, no
 * self-loops).  The CliqueSet stays resident for
 * dpmrf_build_neighborhoods_resident; sizes go to *num_cliques /
 * *num_members (may be NULL). */
dpmrf_status dpmrf_enumerate_maximal_cliques(dpmrf_context* ctx, uint64_t* num_cliques,
                                             uint64_t* num_members);

/* Copy the resident cliques out (offsets: C+1, members: CS; either may be NULL). */
dpmrf_status dpmrf_get_cliques(dpmrf_context* ctx, uint32_t* offsets, uint32_t* members);

/* build_neighborhoods (as dpmrf_build_neighborhoods) from the resident
 * cliques, with no host round trip of the CliqueSet. */
dpmrf_status dpmrf_build_neighborhoods_resident(dpmrf_context* ctx, uint32_t k,
                                                uint64_t* num_slots);

/* ---- the optimization phase -------------------------------------------- */
/* optimize, proj/include/dpmrf/mrf/engine.hpp:99-100 / proj/src/mrf/optimize.cpp:31-74,
 * over the resident graph and neighborhoods.  labels: R entries, mu/sigma:
 * num_labels entries.  opts may be NULL (reference semantics, full trace). */
dpmrf_status dpmrf_optimize(dpmrf_context* ctx, const dpmrf_optimizer_config* config,
                            const dpmrf_run_options* opts, uint32_t* labels, double* mu,
                            double* sigma);

/* optimize(backend, graph, hoods, config) in one call, the exact shape of
 * proj/include/dpmrf/mrf/engine.hpp:99-100: uploads the graph (as
 * dpmrf_set_graph) and the neighborhoods (as dpmrf_set_hoods), then runs
 * dpmrf_optimize -- one host round trip fewer per upload. */
dpmrf_status dpmrf_optimize_arrays(dpmrf_context* ctx, uint32_t num_vertices,
                                   const uint32_t* graph_offsets, const uint32_t* graph_neighbors,
                                   const double* region_mean, uint64_t num_hoods,
                                   const uint32_t* hood_offsets, const uint32_t* hood_members,
                                   const dpmrf_optimizer_config* config,
                                   const dpmrf_run_options* opts, uint32_t* labels, double* mu,
                                   double* sigma);

/* Trace of the last dpmrf_optimize (EmIterationLog / MapIterationLog,
 * engine.hpp:82-99). */
dpmrf_status dpmrf_trace_info(dpmrf_context* ctx, int32_t* em_iters, uint64_t* series);
dpmrf_status dpmrf_trace_em(dpmrf_context* ctx, int32_t em, int32_t* map_iters,
                            double* total_energy, uint8_t* converged, double* mu, double* sigma);
dpmrf_status dpmrf_trace_map(dpmrf_context* ctx, int32_t em, int32_t it, double* hood_energy,
                             uint8_t* converged);
dpmrf_status dpmrf_get_stats(dpmrf_context* ctx, dpmrf_run_stats* out);
/* Caller-owned destination of the full trace (DPMRF_TRACE_FULL) of later
 * optimize calls on ctx: MAP iteration t of EM iteration em lands in row
 * em * map_max_iters + t of hood_energy (f64) and converged (u8), each row
 * `series` values long (dpmrf_trace_info) at a pitch of row_stride values;
 * rows (capacity) must be >= em_max_iters * map_max_iters and row_stride >=
 * the number of hoods, else the call falls back to the library's own
 * buffers.  Rows arrive by DMA while the run proceeds (pinned memory:
 * link-rate copies, no extra host copy); rows t >= the EM's map_iters are
 * unspecified.  NULL detaches.  dpmrf_trace_map keeps working either way.
 * (OptimizeResult.trace, engine.hpp:82-99, optimize.cpp:53-58.) */
dpmrf_status dpmrf_set_trace_sink(dpmrf_context* ctx, double* hood_energy, uint8_t* converged,
                                  uint64_t rows, uint64_t row_stride);

/* ---- step functions (engine.hpp), each on the device -------------------- */
/* init_random, engine.hpp:20-21 / engine.cpp:28-38 (num_labels != 2 ->
 * DPMRF_INPUT_ERROR unless allow_multilabel). */
dpmrf_status dpmrf_init_random(dpmrf_context* ctx, uint32_t num_labels, uint32_t num_vertices,
                               uint64_t seed, int allow_multilabel, double* mu, double* sigma,
                               uint32_t* labels);
/* replicate_by_label, engine.hpp:25-26 / engine.cpp:50-72; outputs M*S each. */
dpmrf_status dpmrf_replicate_by_label(dpmrf_context* ctx, uint32_t num_labels,
                                      uint32_t* test_label, uint32_t* old_index,
                                      uint32_t* hood_id);
/* slot_hood_map, engine.hpp:29-30 / engine.cpp:40-48; S outputs. */
dpmrf_status dpmrf_slot_hood_map(dpmrf_context* ctx, uint32_t* slot_hood);
/* discord_counts, engine.hpp:34-36 / engine.cpp:74-86; M*R outputs. */
dpmrf_status dpmrf_discord_counts(dpmrf_context* ctx, const uint32_t* labels,
                                  uint32_t num_labels, uint32_t* discord);
/* compute_energies, engine.hpp:43-46 / engine.cpp:88-113 over an explicit
 * replicated index of length E (bounds-checked like dpp::gather). */
dpmrf_status dpmrf_compute_energies(dpmrf_context* ctx, uint64_t E, const uint32_t* test_label,
                                    const uint32_t* old_index, uint32_t num_labels,
                                    const double* mu, const double* sigma,
                                    const uint32_t* labels, double beta, double* energies);
/* min_label_energies, engine.hpp:55-56 / engine.cpp:115-145. */
dpmrf_status dpmrf_min_label_energies(dpmrf_context* ctx, uint64_t E, const uint32_t* test_label,
                                      const uint32_t* old_index, const double* energies,
                                      uint64_t num_slots, double* min_energy,
                                      uint32_t* min_label);
/* neighborhood_energy_sums, engine.hpp:60-62 / engine.cpp:147-152: one sum
 * per run of equal adjacent keys; *num_sums receives the run count. */
dpmrf_status dpmrf_neighborhood_energy_sums(dpmrf_context* ctx, uint64_t S,
                                            const uint32_t* slot_hood, const double* min_energy,
                                            double* sums, uint64_t* num_sums);
/* check_convergence, engine.hpp:67-69 / engine.cpp:154-169; history is
 * row-major rows x series, oldest row first. */
dpmrf_status dpmrf_check_convergence(dpmrf_context* ctx, uint64_t rows, uint64_t series,
                                     const double* history, int32_t window, double tol,
                                     uint8_t* flags);
/* update_labels, engine.hpp:75-78 / engine.cpp:171-191 over the resident
 * neighborhoods (argmin: S entries; old/new labels: R entries). */
dpmrf_status dpmrf_update_labels(dpmrf_context* ctx, const uint32_t* argmin_label,
                                 uint32_t num_vertices, const uint32_t* old_labels,
                                 uint32_t* labels);
/* update_parameters, engine.hpp:83-85 / engine.cpp:193-223 over the
 * resident graph's region means. */
dpmrf_status dpmrf_update_parameters(dpmrf_context* ctx, const uint32_t* labels,
                                     uint32_t num_labels, const double* prev_mu,
                                     const double* prev_sigma, double* mu, double* sigma);

/* ---- vertex-range partitioned optimize (one giant slice, config D) --------
 * One region graph split into `world` contiguous vertex ranges (multiples of
 * 256) and as many series ranges; every partition holds the whole static
 * structure (the context's graph + hoods) but computes only its own ranges.
 * Per MAP iteration the partitions exchange the label and minimum-energy
 * halos their neighbors / hoods read and sum the unconverged-hood counters;
 * per EM iteration they allgather the committed labels and the hood-energy
 * row, and every partition runs the same M-step.  Results are bit-identical
 * to dpmrf_optimize on one device (optimize.cpp:31-74).  Trace levels NONE and
 * EM only.
 *   NCCL group: one process per GPU; rank 0 calls dpmrf_nccl_unique_id and
 *     ships the 128 bytes to the others (e.g. torch.distributed), then every
 *     rank calls dpmrf_group_create_nccl with its own context.  libnccl.so.2
 *     is loaded at run time.
 *   Local group: all partitions inside one context on one device, halos moved
 *     by device copies -- the same schedule without NVLink (tests).          */
typedef struct dpmrf_group dpmrf_group;
dpmrf_status dpmrf_nccl_unique_id(uint8_t id[128]);
dpmrf_status dpmrf_group_create_nccl(dpmrf_context* ctx, const uint8_t id[128], int rank,
                                     int world, dpmrf_group** out);
dpmrf_status dpmrf_group_create_local(dpmrf_context* ctx, int world, dpmrf_group** out);
void dpmrf_group_destroy(dpmrf_group* group);
/* Halo statistics of the last partitioned optimize: per-MAP-iteration bytes
 * this rank sends (local group: all partitions), vertex/series range. */
typedef struct dpmrf_group_info {
  int32_t world;
  int32_t rank;              /* -1 for a local group */
  uint32_t vertex_begin, vertex_end;
  uint64_t series_begin, series_end;
  uint64_t halo_bytes_per_map;  /* labels + minima sent per MAP iteration */
  uint64_t gather_bytes_per_em; /* labels + hood row received per EM iteration */
} dpmrf_group_info;
dpmrf_status dpmrf_group_info_get(dpmrf_group* group, dpmrf_group_info* out);
/* Same outputs as dpmrf_optimize on every rank (labels: all R vertices).
 * Stats / EM trace land on the group's context. */
dpmrf_status dpmrf_optimize_partitioned(dpmrf_group* group, const dpmrf_optimizer_config* config,
                                        const dpmrf_run_options* options, uint32_t* labels,
                                        double* mu, double* sigma);

/* ---- diagnostics ---------------------------------------------------------- */
/* The device's correctly rounded natural log used by the device-resident EM
 * loop for log(sigma) (n values, host buffers). */
dpmrf_status dpmrf_debug_log(dpmrf_context* ctx, uint64_t n, const double* x, double* out);

#ifdef __cplusplus
}
#endif
#endif /* DPMRF_CUDA_H */
