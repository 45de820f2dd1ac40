/*
 * dpmrf_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the DPP-PMRF optimization hot path of the reference
 * artifact (/root/reference/proj), used as the parity CHECKER for the CUDA
 * implementation.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library; the product path never does.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 *   (1) the golden vectors of the reference's own tests
 *       (proj/tests/mrf_engine_test.cpp, optimize_test.cpp, cliques_test.cpp), and
 *   (2) the reference itself, compiled from its own sources into oracle/_ref/
 *       by oracle/Makefile, bit for bit on seeded random and phantom inputs.
 *
 * Arithmetic contract (compile with -ffp-contract=off, as proj/CMakeLists.txt:15-18):
 *   energy  = ((x - mu)^2 / two_var + log_sigma) + beta * discord   (model.hpp:66-72)
 *   folds   = 1024-element leaves folded left to right, leaf partials combined
 *             by a pairwise tree split at bit_floor(n-1)          (kernels.hpp:20-65)
 *
 * Every function cites the reference lines it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_INPUT_ERROR 1
#define ORC_INVALID_ARGUMENT 2
#define ORC_OUT_OF_RANGE 3
#define ORC_NOMEM 6

#define ORC_LEAF 1024u          /* kFoldLeafSize, kernels.hpp:27 */
#define ORC_SIGMA_FLOOR 1e-3    /* kSigmaFloor, model.hpp:9 */

/* ------------------------------------------------------------------ */
/* SplitMix64 stream, engine.cpp:15-24                                  */
/* ------------------------------------------------------------------ */
static uint64_t orc_next_u64(uint64_t *state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static double orc_next_unit(uint64_t *state) {
  return (double)(orc_next_u64(state) >> 11) * 0x1.0p-53;
}

/* init_random, engine.cpp:28-38.  The reference rejects M != 2
 * (engine.cpp:30); allow_multilabel != 0 applies the same draw order to any
 * M (the documented M=5 extension). */
int orc_init_random(uint32_t M, uint32_t R, uint64_t seed, int allow_multilabel, double *mu,
                    double *sigma, uint32_t *labels) {
  if (M != 2 && !(allow_multilabel && M >= 1)) return ORC_INPUT_ERROR;
  uint64_t state = seed;
  for (uint32_t l = 0; l < M; ++l) mu[l] = 255.0 * orc_next_unit(&state);
  for (uint32_t l = 0; l < M; ++l) {
    double s = 255.0 * orc_next_unit(&state);
    sigma[l] = s < ORC_SIGMA_FLOOR ? ORC_SIGMA_FLOOR : s; /* std::max(s, floor) */
  }
  for (uint32_t v = 0; v < R; ++v) labels[v] = (uint32_t)(orc_next_u64(&state) % M);
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Fixed fold topology, kernels.hpp:37-65                               */
/* ------------------------------------------------------------------ */
static double fold_leaf_add(const double *x, size_t n) {
  double acc = x[0];
  for (size_t i = 1; i < n; ++i) acc = acc + x[i];
  return acc;
}

static double fold_tree_add(const double *p, size_t count) {
  if (count == 1) return p[0];
  size_t split = 1;
  while (split * 2 <= count - 1) split *= 2; /* std::bit_floor(count - 1) */
  double left = fold_tree_add(p, split);
  double right = fold_tree_add(p + split, count - split);
  return left + right;
}

/* fold_range<plus>, kernels.hpp:56-65 (n >= 1). */
double orc_fold_range_add(const double *x, size_t n) {
  if (n <= ORC_LEAF) return fold_leaf_add(x, n);
  size_t leaves = (n + ORC_LEAF - 1) / ORC_LEAF;
  double *partials = (double *)malloc(leaves * sizeof(double));
  for (size_t k = 0; k < leaves; ++k) {
    size_t b = k * ORC_LEAF;
    size_t e = b + ORC_LEAF < n ? b + ORC_LEAF : n;
    partials[k] = fold_leaf_add(x + b, e - b);
  }
  double r = fold_tree_add(partials, leaves);
  free(partials);
  return r;
}

/* fold_tree<plus> over given leaf partials (kernels.hpp:45-51), count >= 1:
 * the combine step of a fold whose leaves were folded elsewhere. */
double orc_fold_tree_add(const double *p, size_t count) { return fold_tree_add(p, count); }

/* dpp::reduce<plus> with identity 0.0, kernels.hpp:124-139. */
double orc_reduce_add(const double *x, size_t n) {
  if (n == 0) return 0.0;
  return orc_fold_range_add(x, n);
}

/* (energy, label) pair folded with the keep-strictly-smaller op of
 * min_label_energies, engine.cpp:123-127. */
typedef struct {
  double e;
  uint32_t l;
} orc_el;

static orc_el el_op(orc_el a, orc_el b) { return b.e < a.e ? b : a; }

static orc_el fold_leaf_el(const orc_el *x, size_t n) {
  orc_el acc = x[0];
  for (size_t i = 1; i < n; ++i) acc = el_op(acc, x[i]);
  return acc;
}

static orc_el fold_tree_el(const orc_el *p, size_t count) {
  if (count == 1) return p[0];
  size_t split = 1;
  while (split * 2 <= count - 1) split *= 2;
  orc_el left = fold_tree_el(p, split);
  orc_el right = fold_tree_el(p + split, count - split);
  return el_op(left, right);
}

static orc_el fold_range_el(const orc_el *x, size_t n) {
  if (n <= ORC_LEAF) return fold_leaf_el(x, n);
  size_t leaves = (n + ORC_LEAF - 1) / ORC_LEAF;
  orc_el *partials = (orc_el *)malloc(leaves * sizeof(orc_el));
  for (size_t k = 0; k < leaves; ++k) {
    size_t b = k * ORC_LEAF;
    size_t e = b + ORC_LEAF < n ? b + ORC_LEAF : n;
    partials[k] = fold_leaf_el(x + b, e - b);
  }
  orc_el r = fold_tree_el(partials, leaves);
  free(partials);
  return r;
}

/* ------------------------------------------------------------------ */
/* Replication layout, engine.cpp:40-72                                 */
/* ------------------------------------------------------------------ */
void orc_slot_hood_map(uint64_t H, const uint32_t *hood_off, uint32_t *slot_hood) {
  for (uint64_t h = 0; h < H; ++h)
    for (uint32_t s = hood_off[h]; s < hood_off[h + 1]; ++s) slot_hood[s] = (uint32_t)h;
}

/* e = M*o + l*sz + j, engine.cpp:59-70 */
void orc_replicate_by_label(uint64_t H, const uint32_t *hood_off, uint32_t M,
                            uint32_t *test_label, uint32_t *old_index, uint32_t *hood_id) {
  for (uint64_t h = 0; h < H; ++h) {
    uint64_t o = hood_off[h], sz = hood_off[h + 1] - hood_off[h];
    for (uint64_t j = 0; j < sz; ++j)
      for (uint32_t l = 0; l < M; ++l) {
        uint64_t e = (uint64_t)M * o + (uint64_t)l * sz + j;
        test_label[e] = l;
        old_index[e] = (uint32_t)(o + j);
        hood_id[e] = (uint32_t)h;
      }
  }
}

/* discord[l*R+v] = #{u in adj(v) : labels[u] != l}, engine.cpp:74-86 */
void orc_discord_counts(uint32_t R, const uint32_t *g_off, const uint32_t *g_nbr,
                        const uint32_t *labels, uint32_t M, uint32_t *discord) {
  for (uint32_t l = 0; l < M; ++l)
    for (uint32_t v = 0; v < R; ++v) {
      uint32_t c = 0;
      for (uint32_t a = g_off[v]; a < g_off[v + 1]; ++a) c += labels[g_nbr[a]] != l;
      discord[(uint64_t)l * R + v] = c;
    }
}

/* make_label_terms, model.hpp:48-60 (std::log from the host libm). */
void orc_label_terms(uint32_t M, const double *mu, const double *sigma, double *t_mu,
                     double *t_two_var, double *t_log_sigma) {
  for (uint32_t l = 0; l < M; ++l) {
    t_mu[l] = mu[l];
    t_two_var[l] = 2.0 * (sigma[l] * sigma[l]);
    t_log_sigma[l] = log(sigma[l]);
  }
}

/* label_energy, model.hpp:66-72 -- fixed order sub, mul, div, add, mul, add. */
static double orc_label_energy(double x, double mu, double two_var, double log_sigma,
                               double beta, uint32_t discord) {
  const double d = x - mu;
  const double q = (d * d) / two_var;
  const double data_term = q + log_sigma;
  return data_term + beta * (double)discord;
}

double orc_label_energy_pub(double x, double mu, double two_var, double log_sigma, double beta,
                            uint32_t discord) {
  return orc_label_energy(x, mu, two_var, log_sigma, beta, discord);
}

/* compute_energies, engine.cpp:88-113 (gathers bounds-checked as
 * dpp::gather, kernels.hpp:306-318 -> std::out_of_range). */
int orc_compute_energies(uint32_t R, const uint32_t *g_off, const uint32_t *g_nbr,
                         const double *mean, uint64_t S, const uint32_t *members, uint64_t E,
                         const uint32_t *test_label, const uint32_t *old_index, uint32_t M,
                         const double *mu, const double *sigma, const uint32_t *labels,
                         double beta, double *out) {
  double *t_mu = (double *)malloc(M * sizeof(double) + 1);
  double *t_tv = (double *)malloc(M * sizeof(double) + 1);
  double *t_ls = (double *)malloc(M * sizeof(double) + 1);
  uint32_t *disc = (uint32_t *)malloc((uint64_t)M * R * sizeof(uint32_t) + 1);
  int rc = ORC_OK;
  orc_label_terms(M, mu, sigma, t_mu, t_tv, t_ls);
  orc_discord_counts(R, g_off, g_nbr, labels, M, disc);
  for (uint64_t e = 0; e < E && rc == ORC_OK; ++e) {
    if (old_index[e] >= S) { rc = ORC_OUT_OF_RANGE; break; }
    uint32_t v = members[old_index[e]];
    uint32_t l = test_label[e];
    if (v >= R || l >= M) { rc = ORC_OUT_OF_RANGE; break; }
    out[e] = orc_label_energy(mean[v], t_mu[l], t_tv[l], t_ls[l], beta, disc[(uint64_t)l * R + v]);
  }
  free(t_mu); free(t_tv); free(t_ls); free(disc);
  return rc;
}

/* Stable counting sort of positions by a u32 key (the unique stable order
 * of sort_by_key, kernels.hpp:255-303).  perm[i] = position of the i-th
 * element in key order; key_start has nkeys+1 entries. */
static int stable_order(uint64_t n, const uint32_t *keys, uint32_t nkeys, uint64_t *perm,
                        uint64_t *key_start) {
  memset(key_start, 0, (nkeys + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) {
    if (keys[i] >= nkeys) return ORC_OUT_OF_RANGE;
    key_start[keys[i] + 1]++;
  }
  for (uint32_t k = 0; k < nkeys; ++k) key_start[k + 1] += key_start[k];
  uint64_t *fill = (uint64_t *)malloc((nkeys + 1) * sizeof(uint64_t));
  memcpy(fill, key_start, (nkeys + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) perm[fill[keys[i]]++] = i;
  free(fill);
  return ORC_OK;
}

/* min_label_energies, engine.cpp:115-145: stable sort by old_index, keyed
 * fold_range with the keep-strictly-smaller op, scatter into num_slots
 * outputs pre-filled with (0.0, 0).  Keys >= num_slots would be an
 * out-of-range scatter (kernels.hpp:337). */
int orc_min_label_energies(uint64_t E, const uint32_t *test_label, const uint32_t *old_index,
                           const double *energies, uint64_t num_slots, double *out_e,
                           uint32_t *out_l) {
  for (uint64_t s = 0; s < num_slots; ++s) { out_e[s] = 0.0; out_l[s] = 0; }
  if (E == 0) return ORC_OK;
  uint32_t maxk = 0;
  for (uint64_t e = 0; e < E; ++e) if (old_index[e] > maxk) maxk = old_index[e];
  if (maxk >= num_slots) return ORC_OUT_OF_RANGE;
  uint64_t *perm = (uint64_t *)malloc(E * sizeof(uint64_t));
  uint64_t *ks = (uint64_t *)malloc((maxk + 2) * sizeof(uint64_t));
  stable_order(E, old_index, maxk + 1, perm, ks);
  orc_el *run = (orc_el *)malloc(E * sizeof(orc_el));
  for (uint32_t k = 0; k <= maxk; ++k) {
    uint64_t lo = ks[k], hi = ks[k + 1];
    if (lo == hi) continue;
    for (uint64_t i = lo; i < hi; ++i) {
      run[i - lo].e = energies[perm[i]];
      run[i - lo].l = test_label[perm[i]];
    }
    orc_el r = fold_range_el(run, hi - lo);
    out_e[k] = r.e;
    out_l[k] = r.l;
  }
  free(perm); free(ks); free(run);
  return ORC_OK;
}

/* neighborhood_energy_sums, engine.cpp:147-152: reduce_by_key<plus> over
 * runs of equal adjacent keys (kernels.hpp:226-253).  Returns the run count
 * through *num_out (one output per run, NOT per hood id). */
void orc_neighborhood_energy_sums(uint64_t S, const uint32_t *slot_hood, const double *min_e,
                                  double *out, uint64_t *num_out) {
  uint64_t runs = 0, lo = 0;
  while (lo < S) {
    uint64_t hi = lo + 1;
    while (hi < S && slot_hood[hi] == slot_hood[lo]) ++hi;
    out[runs++] = orc_fold_range_add(min_e + lo, hi - lo);
    lo = hi;
  }
  *num_out = runs;
}

/* check_convergence, engine.cpp:154-169.  history is row-major
 * (rows x series), oldest row first. */
void orc_check_convergence(uint64_t rows, uint64_t series, const double *history, int window,
                           double tol, uint8_t *out) {
  if (rows < (uint64_t)window + 1) {
    for (uint64_t c = 0; c < series; ++c) out[c] = 0;
    return;
  }
  const double *last = history + (rows - 1) * series;
  for (uint64_t c = 0; c < series; ++c) {
    uint8_t ok = 1;
    for (int i = 1; i <= window; ++i) {
      const double prev = history[(rows - 1 - (uint64_t)i) * series + c];
      if (!(fabs(last[c] - prev) < tol)) { ok = 0; break; }
    }
    out[c] = ok;
  }
}

/* update_labels, engine.cpp:171-191: stable sort of slots by vertex, keep the
 * first (lowest-hood) slot, scatter; uncovered vertices keep old labels. */
int orc_update_labels(uint64_t S, const uint32_t *members, const uint32_t *argmin, uint32_t R,
                      const uint32_t *old_labels, uint32_t *out) {
  for (uint32_t v = 0; v < R; ++v) out[v] = old_labels[v];
  if (S == 0) return ORC_OK;
  uint8_t *seen = (uint8_t *)calloc(R + 1, 1);
  int rc = ORC_OK;
  for (uint64_t s = 0; s < S; ++s) {
    uint32_t v = members[s];
    if (v >= R) { rc = ORC_OUT_OF_RANGE; break; }
    if (!seen[v]) { seen[v] = 1; out[v] = argmin[s]; }
  }
  free(seen);
  return rc;
}

/* update_parameters, engine.cpp:193-223: stable sort by label, keyed
 * fold_range sums, mu = sum/n, then fold_range of (x-mu)^2, sigma =
 * max(sqrt(sq/n), floor); empty labels keep previous parameters. */
int orc_update_parameters(uint32_t R, const double *mean, const uint32_t *labels, uint32_t M,
                          const double *prev_mu, const double *prev_sigma, double *mu,
                          double *sigma) {
  for (uint32_t l = 0; l < M; ++l) { mu[l] = prev_mu[l]; sigma[l] = prev_sigma[l]; }
  if (R == 0) return ORC_OK;
  uint32_t maxl = 0;
  for (uint32_t v = 0; v < R; ++v) if (labels[v] > maxl) maxl = labels[v];
  if (maxl >= M) return ORC_INVALID_ARGUMENT; /* engine.cpp:206-208 */
  uint64_t *perm = (uint64_t *)malloc((uint64_t)R * sizeof(uint64_t));
  uint64_t *ks = (uint64_t *)malloc((M + 1) * sizeof(uint64_t));
  double *x = (double *)malloc((uint64_t)R * sizeof(double));
  stable_order(R, labels, M, perm, ks);
  for (uint32_t l = 0; l < M; ++l) {
    uint64_t lo = ks[l], hi = ks[l + 1];
    if (lo == hi) continue;
    for (uint64_t i = lo; i < hi; ++i) x[i - lo] = mean[perm[i]];
    const double n = (double)(uint32_t)(hi - lo);
    mu[l] = orc_fold_range_add(x, hi - lo) / n;
    for (uint64_t i = 0; i < hi - lo; ++i) {
      const double d = x[i] - mu[l];
      x[i] = d * d;
    }
    const double sd = sqrt(orc_fold_range_add(x, hi - lo) / n);
    sigma[l] = sd < ORC_SIGMA_FLOOR ? ORC_SIGMA_FLOOR : sd;
  }
  free(perm); free(ks); free(x);
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* build_neighborhoods, neighborhoods.cpp:10-57                         */
/* ------------------------------------------------------------------ */
static int cmp_u32(const void *a, const void *b) {
  uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  return x < y ? -1 : (x > y);
}

/* Two-call form: with members == NULL only fills *num_slots. hood_off gets
 * C+1 entries; source_clique C entries (identity, neighborhoods.cpp:53-55). */
int orc_build_neighborhoods(uint32_t R, const uint32_t *g_off, const uint32_t *g_nbr, uint64_t C,
                            const uint32_t *c_off, const uint32_t *c_mem, uint32_t k,
                            uint32_t *hood_off, uint32_t *members, uint32_t *source_clique,
                            uint64_t *num_slots) {
  if (k != 1) return ORC_INPUT_ERROR; /* neighborhoods.cpp:12 */
  uint64_t total = 0, cap = 0;
  uint32_t *buf = NULL;
  if (hood_off) hood_off[0] = 0;
  for (uint64_t c = 0; c < C; ++c) {
    uint64_t cnt = 0;
    for (uint32_t s = c_off[c]; s < c_off[c + 1]; ++s) {
      if (c_mem[s] >= R) { free(buf); return ORC_OUT_OF_RANGE; }
      cnt += 1 + (g_off[c_mem[s] + 1] - g_off[c_mem[s]]);
    }
    if (cnt > cap) { cap = cnt * 2; buf = (uint32_t *)realloc(buf, cap * sizeof(uint32_t)); }
    uint64_t n = 0;
    for (uint32_t s = c_off[c]; s < c_off[c + 1]; ++s) {
      uint32_t m = c_mem[s];
      buf[n++] = m;
      for (uint32_t a = g_off[m]; a < g_off[m + 1]; ++a) buf[n++] = g_nbr[a];
    }
    qsort(buf, n, sizeof(uint32_t), cmp_u32);
    uint64_t u = 0;
    for (uint64_t i = 0; i < n; ++i)
      if (i == 0 || buf[i] != buf[i - 1]) {
        if (members) members[total + u] = buf[i];
        ++u;
      }
    total += u;
    if (hood_off) hood_off[c + 1] = (uint32_t)total;
    if (source_clique) source_clique[c] = (uint32_t)c;
  }
  free(buf);
  *num_slots = total;
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* optimize, optimize.cpp:13-74 (DPP-engine semantics)                  */
/* ------------------------------------------------------------------ */
typedef struct {
  uint32_t num_labels;
  int32_t em_max_iters;
  int32_t map_max_iters;
  int32_t convergence_window;
  double convergence_tol;
  double beta;
  uint64_t rng_seed;
} orc_config;

/* validate_config, optimize.cpp:13-23 (num_labels check relaxed under the
 * multilabel extension). */
int orc_validate_config(const orc_config *c, int allow_multilabel) {
  if (c->num_labels != 2 && !(allow_multilabel && c->num_labels >= 1)) return ORC_INPUT_ERROR;
  if (c->em_max_iters < 0) return ORC_INPUT_ERROR;
  if (c->map_max_iters < 1) return ORC_INPUT_ERROR;
  if (c->convergence_window < 1) return ORC_INPUT_ERROR;
  if (c->convergence_window >= c->map_max_iters) return ORC_INPUT_ERROR;
  if (!(c->convergence_tol > 0.0)) return ORC_INPUT_ERROR;
  if (!(c->beta >= 0.0)) return ORC_INPUT_ERROR;
  return ORC_OK;
}

/* Trace buffers (caller-allocated, sized for the worst case):
 *   em_map_iters[em], em_total[em], em_conv[em], em_mu[em*M+l], em_sigma[em*M+l]
 *   map_energy[(em*map_max + it)*H + h] and map_conv[...] (may be NULL).
 * fixed_work != 0 removes the two early exits (optimize.cpp:59, :71), the
 * fixed-work workload of BASELINE.md; flags are still computed and logged. */
typedef struct {
  int32_t *em_map_iters;
  double *em_total;
  uint8_t *em_conv;
  double *em_mu;
  double *em_sigma;
  double *map_energy;
  uint8_t *map_conv;
  int32_t em_iters;   /* out */
  uint64_t series;    /* out: hood-energy series length (runs of slot_hood) */
} orc_trace;

static int all_set(const uint8_t *f, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) if (!f[i]) return 0;
  return 1;
}

int orc_optimize(uint32_t R, const uint32_t *g_off, const uint32_t *g_nbr, const double *mean,
                 uint64_t H, const uint32_t *hood_off, const uint32_t *members,
                 const orc_config *cfg, int fixed_work, int allow_multilabel, uint32_t *labels,
                 double *mu, double *sigma, orc_trace *tr) {
  int rc = orc_validate_config(cfg, allow_multilabel);
  if (rc) return rc;
  const uint32_t M = cfg->num_labels;
  rc = orc_init_random(M, R, cfg->rng_seed, allow_multilabel, mu, sigma, labels);
  if (rc) return rc;
  tr->em_iters = 0;
  tr->series = 0;
  if (cfg->em_max_iters == 0) return ORC_OK;

  const uint64_t S = hood_off[H];
  const int L = cfg->convergence_window;
  uint32_t *slot_hood = (uint32_t *)malloc(S * sizeof(uint32_t) + 4);
  double *slot_min = (double *)malloc(S * sizeof(double) + 8);
  uint32_t *slot_arg = (uint32_t *)malloc(S * sizeof(uint32_t) + 4);
  uint32_t *disc = (uint32_t *)malloc((uint64_t)M * R * sizeof(uint32_t) + 4);
  uint32_t *next = (uint32_t *)malloc((uint64_t)R * sizeof(uint32_t) + 4);
  double *hist = (double *)malloc((uint64_t)cfg->map_max_iters * (H + 1) * sizeof(double));
  uint8_t *flags = (uint8_t *)malloc(H + 1);
  double *em_hist = (double *)malloc(((uint64_t)cfg->em_max_iters + 1) * sizeof(double));
  double t_mu[256], t_tv[256], t_ls[256];
  double nmu[256], nsig[256];
  orc_slot_hood_map(H, hood_off, slot_hood);

  for (uint64_t s = 0; s < S; ++s)
    if (members[s] >= R) { rc = ORC_OUT_OF_RANGE; goto done; }

  for (int em = 0; em < cfg->em_max_iters; ++em) {
    orc_label_terms(M, mu, sigma, t_mu, t_tv, t_ls);
    uint64_t series = 0;
    int it = 0;
    for (; it < cfg->map_max_iters; ++it) {
      /* compute_energies + min_label_energies: per slot, the min over the
       * label-ordered replicas (label-major layout, engine.cpp:59-70). */
      orc_discord_counts(R, g_off, g_nbr, labels, M, disc);
      for (uint64_t s = 0; s < S; ++s) {
        const uint32_t v = members[s];
        orc_el acc = {0.0, 0};
        for (uint32_t l = 0; l < M; ++l) {
          orc_el c;
          c.e = orc_label_energy(mean[v], t_mu[l], t_tv[l], t_ls[l], cfg->beta,
                                 disc[(uint64_t)l * R + v]);
          c.l = l;
          acc = l == 0 ? c : el_op(acc, c);
        }
        slot_min[s] = acc.e;
        slot_arg[s] = acc.l;
      }
      orc_update_labels(S, members, slot_arg, R, labels, next);
      memcpy(labels, next, (uint64_t)R * sizeof(uint32_t));
      double *row = hist + (uint64_t)it * (H + 1);
      orc_neighborhood_energy_sums(S, slot_hood, slot_min, row, &series);
      /* check_convergence (engine.cpp:154-169) over history rows strided by H+1. */
      {
        if ((uint64_t)it + 1 < (uint64_t)L + 1) {
          memset(flags, 0, series);
        } else {
          for (uint64_t c = 0; c < series; ++c) {
            uint8_t ok = 1;
            for (int i = 1; i <= L; ++i) {
              const double prev = hist[(uint64_t)(it - i) * (H + 1) + c];
              if (!(fabs(row[c] - prev) < cfg->convergence_tol)) { ok = 0; break; }
            }
            flags[c] = ok;
          }
        }
      }
      if (tr->map_energy) {
        memcpy(tr->map_energy + ((uint64_t)em * cfg->map_max_iters + it) * H, row,
               series * sizeof(double));
        memcpy(tr->map_conv + ((uint64_t)em * cfg->map_max_iters + it) * H, flags, series);
      }
      const int done = all_set(flags, series);
      if (done && !fixed_work) { ++it; break; }
    }
    if (it > cfg->map_max_iters) it = cfg->map_max_iters;
    tr->series = series;
    rc = orc_update_parameters(R, mean, labels, M, mu, sigma, nmu, nsig);
    if (rc) goto done;
    memcpy(mu, nmu, M * sizeof(double));
    memcpy(sigma, nsig, M * sizeof(double));
    const double total = orc_reduce_add(hist + (uint64_t)(it - 1) * (H + 1), series);
    em_hist[em] = total;
    uint8_t conv = 0;
    if (em + 1 >= L + 1) {
      conv = 1;
      for (int i = 1; i <= L; ++i)
        if (!(fabs(total - em_hist[em - i]) < cfg->convergence_tol)) { conv = 0; break; }
    }
    tr->em_map_iters[em] = it;
    tr->em_total[em] = total;
    tr->em_conv[em] = conv;
    memcpy(tr->em_mu + (uint64_t)em * M, mu, M * sizeof(double));
    memcpy(tr->em_sigma + (uint64_t)em * M, sigma, M * sizeof(double));
    tr->em_iters = em + 1;
    if (conv && !fixed_work) break;
  }
done:
  free(slot_hood); free(slot_min); free(slot_arg); free(disc); free(next);
  free(hist); free(flags); free(em_hist);
  return rc;
}

/* optimize_reference, optimize.cpp:76-144: Gauss-Seidel sweep over hoods in
 * index order, committing each hood's winners immediately.  The T* CPU
 * baseline and the <=5% energy-gap cross-check (acceptance.cpp:428-445);
 * NOT the label-parity oracle. Trace: em_* arrays only. */
int orc_optimize_reference(uint32_t R, const uint32_t *g_off, const uint32_t *g_nbr,
                           const double *mean, uint64_t H, const uint32_t *hood_off,
                           const uint32_t *members, const orc_config *cfg, int fixed_work,
                           int allow_multilabel, uint32_t *labels, double *mu, double *sigma,
                           orc_trace *tr) {
  int rc = orc_validate_config(cfg, allow_multilabel);
  if (rc) return rc;
  const uint32_t M = cfg->num_labels;
  rc = orc_init_random(M, R, cfg->rng_seed, allow_multilabel, mu, sigma, labels);
  if (rc) return rc;
  tr->em_iters = 0;
  tr->series = H;
  if (cfg->em_max_iters == 0) return ORC_OK;
  const int L = cfg->convergence_window;
  double *hist = (double *)malloc((uint64_t)cfg->map_max_iters * (H + 1) * sizeof(double));
  double *em_hist = (double *)malloc(((uint64_t)cfg->em_max_iters + 1) * sizeof(double));
  uint32_t *win = NULL;
  uint64_t wcap = 0;
  double t_mu[256], t_tv[256], t_ls[256], nmu[256], nsig[256];
  for (int em = 0; em < cfg->em_max_iters; ++em) {
    orc_label_terms(M, mu, sigma, t_mu, t_tv, t_ls);
    int it = 0;
    for (; it < cfg->map_max_iters; ++it) {
      double *row = hist + (uint64_t)it * (H + 1);
      for (uint64_t h = 0; h < H; ++h) {
        const uint32_t lo = hood_off[h], hi = hood_off[h + 1];
        if (hi - lo > wcap) { wcap = 2 * (uint64_t)(hi - lo); win = (uint32_t *)realloc(win, wcap * 4); }
        double sum = 0.0;
        for (uint32_t s = lo; s < hi; ++s) {
          const uint32_t v = members[s];
          double best = 0.0;
          uint32_t best_l = 0;
          for (uint32_t l = 0; l < M; ++l) {
            uint32_t dc = 0;
            for (uint32_t a = g_off[v]; a < g_off[v + 1]; ++a) dc += labels[g_nbr[a]] != l;
            const double e = orc_label_energy(mean[v], t_mu[l], t_tv[l], t_ls[l], cfg->beta, dc);
            if (l == 0 || e < best) { best = e; best_l = l; }
          }
          win[s - lo] = best_l;
          sum = s == lo ? best : sum + best;
        }
        for (uint32_t s = lo; s < hi; ++s) labels[members[s]] = win[s - lo];
        row[h] = sum;
      }
      int done = 0;
      if (it + 1 >= L + 1) {
        done = 1;
        for (uint64_t c = 0; c < H && done; ++c)
          for (int i = 1; i <= L; ++i)
            if (!(fabs(row[c] - hist[(uint64_t)(it - i) * (H + 1) + c]) < cfg->convergence_tol)) {
              done = 0;
              break;
            }
      } else if (H == 0) {
        done = 1;
      }
      if (done && !fixed_work) { ++it; break; }
    }
    if (it > cfg->map_max_iters) it = cfg->map_max_iters;
    rc = orc_update_parameters(R, mean, labels, M, mu, sigma, nmu, nsig);
    if (rc) break;
    memcpy(mu, nmu, M * sizeof(double));
    memcpy(sigma, nsig, M * sizeof(double));
    const double total = orc_reduce_add(hist + (uint64_t)(it - 1) * (H + 1), H);
    em_hist[em] = total;
    uint8_t conv = 0;
    if (em + 1 >= L + 1) {
      conv = 1;
      for (int i = 1; i <= L; ++i)
        if (!(fabs(total - em_hist[em - i]) < cfg->convergence_tol)) { conv = 0; break; }
    }
    tr->em_map_iters[em] = it;
    tr->em_total[em] = total;
    tr->em_conv[em] = conv;
    memcpy(tr->em_mu + (uint64_t)em * M, mu, M * sizeof(double));
    memcpy(tr->em_sigma + (uint64_t)em * M, sigma, M * sizeof(double));
    tr->em_iters = em + 1;
    if (conv && !fixed_work) break;
  }
  free(hist); free(em_hist); free(win);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Evaluation.                                 */
/* ------------------------------------------------------------------ */
/* confusion_u8, scalar_kernels.cpp:48-63 (behind confusion(),
 * metrics.cpp:8-14): nonzero = positive; counts = {tp, tn, fp, fn}. */
void orc_confusion(uint64_t n, const uint8_t *pred, const uint8_t *truth, uint64_t counts[4]) {
  uint64_t tp = 0, tn = 0, fp = 0, fn = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const int p = pred[i] != 0, t = truth[i] != 0;
    tp += p && t;
    tn += !p && !t;
    fp += p && !t;
    fn += !p && t;
  }
  counts[0] = tp;
  counts[1] = tn;
  counts[2] = fp;
  counts[3] = fn;
}

/* The segment write-back, tools/main.cpp:157-165 (acceptance.cpp:359-370):
 * the darker class (mu[0] <= mu[1] ? 0 : 1) is the pore phase; mask[p] =
 * labels[region[p]] == pore. */
void orc_labels_to_mask(uint64_t n, const uint32_t *region, const uint32_t *labels,
                        const double *mu, uint8_t *mask) {
  const uint32_t pore = mu[0] <= mu[1] ? 0u : 1u;
  for (uint64_t i = 0; i < n; ++i) mask[i] = labels[region[i]] == pore ? 1 : 0;
}

/* validate_label_map, label_map.cpp:38-78: serial union-find over same-id
 * right / down pixel pairs (:60-67), roots compared per region in scan order
 * (:68-76).  Returns 0 and *num_regions, or INPUT_ERROR with *detail = the
 * lowest unused id (*kind = 1) or the region that is not 4-connected
 * (*kind = 2); *kind = 3 for an empty map. */
static uint32_t uf_find(uint32_t *p, uint32_t x) {
  while (p[x] != x) {
    p[x] = p[p[x]];
    x = p[x];
  }
  return x;
}

int orc_validate_label_map(uint32_t w, uint32_t h, const uint32_t *region, uint32_t *num_regions,
                           int *kind, uint32_t *detail) {
  const uint64_t n = (uint64_t)w * h;
  *kind = 0;
  if (n == 0) {
    *kind = 3;
    return ORC_INPUT_ERROR;
  }
  uint32_t max_id = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (region[i] > max_id) max_id = region[i];
  const uint64_t num = (uint64_t)max_id + 1;
  uint8_t *used = (uint8_t *)calloc(num, 1);
  uint32_t *parent = (uint32_t *)malloc(n * sizeof(uint32_t));
  uint32_t *root_of = (uint32_t *)malloc(num * sizeof(uint32_t));
  int rc = 0;
  if (!used || !parent || !root_of) {
    rc = ORC_NOMEM;
    goto done;
  }
  for (uint64_t i = 0; i < n; ++i) used[region[i]] = 1;
  for (uint64_t id = 0; id < num; ++id)
    if (!used[id]) {
      *kind = 1;
      *detail = (uint32_t)id;
      rc = ORC_INPUT_ERROR;
      goto done;
    }
  for (uint64_t i = 0; i < n; ++i) parent[i] = (uint32_t)i;
  for (uint32_t y = 0; y < h; ++y)
    for (uint32_t x = 0; x < w; ++x) {
      const uint64_t i = (uint64_t)y * w + x;
      if (x + 1 < w && region[i] == region[i + 1]) {
        const uint32_t a = uf_find(parent, (uint32_t)i), b = uf_find(parent, (uint32_t)(i + 1));
        if (a != b) parent[b] = a;
      }
      if (y + 1 < h && region[i] == region[i + w]) {
        const uint32_t a = uf_find(parent, (uint32_t)i), b = uf_find(parent, (uint32_t)(i + w));
        if (a != b) parent[b] = a;
      }
    }
  for (uint64_t id = 0; id < num; ++id) root_of[id] = 0xFFFFFFFFu;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t id = region[i], r = uf_find(parent, (uint32_t)i);
    if (root_of[id] == 0xFFFFFFFFu) {
      root_of[id] = r;
    } else if (root_of[id] != r) {
      *kind = 2;
      *detail = id;
      rc = ORC_INPUT_ERROR;
      goto done;
    }
  }
  *num_regions = (uint32_t)num;
done:
  free(used);
  free(parent);
  free(root_of);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Structure builders.                      */
/* Outputs of variable length are malloc'd; release with orc_free.      */
/* ------------------------------------------------------------------ */
void orc_free(void *p) { free(p); }

static int cmp_u64(const void *a, const void *b) {
  const uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* build_region_graph, region_graph.cpp:10-73: directed (a,b) and (b,a) keys
 * for every right / down pixel pair in different regions (:21-38), sorted,
 * uniqued (:40-42), split by source into the CSR (:44-53); region sizes and
 * integer intensity sums divided once per region (:57-71).  R == 0 ->
 * INPUT_ERROR (:14); an id >= R -> OUT_OF_RANGE; an unused id (map not
 * validated) -> INPUT_ERROR. */
int orc_region_graph(uint32_t w, uint32_t h, const uint8_t *px, const uint32_t *reg, uint32_t R,
                     uint32_t *off, uint32_t **nbr_out, uint64_t *A_out, double *mean,
                     uint32_t *size) {
  const uint64_t n = (uint64_t)w * h;
  *nbr_out = NULL;
  *A_out = 0;
  if (R == 0) return ORC_INPUT_ERROR;
  for (uint64_t i = 0; i < n; ++i)
    if (reg[i] >= R) return ORC_OUT_OF_RANGE;
  uint64_t cnt = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t x = (uint32_t)(i % w);
    if (x + 1 < w && reg[i] != reg[i + 1]) cnt += 2;
    if (i + w < n && reg[i] != reg[i + w]) cnt += 2;
  }
  uint64_t *keys = (uint64_t *)malloc((cnt ? cnt : 1) * sizeof(uint64_t));
  uint64_t *sum = (uint64_t *)calloc(R, sizeof(uint64_t));
  if (!keys || !sum) {
    free(keys);
    free(sum);
    return ORC_NOMEM;
  }
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t x = (uint32_t)(i % w);
    if (x + 1 < w && reg[i] != reg[i + 1]) {
      keys[k++] = ((uint64_t)reg[i] << 32) | reg[i + 1];
      keys[k++] = ((uint64_t)reg[i + 1] << 32) | reg[i];
    }
    if (i + w < n && reg[i] != reg[i + w]) {
      keys[k++] = ((uint64_t)reg[i] << 32) | reg[i + w];
      keys[k++] = ((uint64_t)reg[i + w] << 32) | reg[i];
    }
  }
  qsort(keys, cnt, sizeof(uint64_t), cmp_u64);
  uint64_t A = 0;
  for (uint64_t i = 0; i < cnt; ++i)
    if (i == 0 || keys[i] != keys[i - 1]) keys[A++] = keys[i];
  uint32_t *nbr = (uint32_t *)malloc((A ? A : 1) * sizeof(uint32_t));
  if (!nbr) {
    free(keys);
    free(sum);
    return ORC_NOMEM;
  }
  memset(off, 0, ((size_t)R + 1) * sizeof(uint32_t));
  for (uint64_t i = 0; i < A; ++i) {
    nbr[i] = (uint32_t)keys[i];
    off[(keys[i] >> 32) + 1] += 1;
  }
  for (uint32_t v = 0; v < R; ++v) off[v + 1] += off[v];
  memset(size, 0, (size_t)R * sizeof(uint32_t));
  for (uint64_t i = 0; i < n; ++i) {
    size[reg[i]] += 1;
    sum[reg[i]] += px[i];
  }
  int rc = ORC_OK;
  for (uint32_t r = 0; r < R; ++r) {
    if (size[r] == 0) rc = ORC_INPUT_ERROR;
    mean[r] = size[r] ? (double)sum[r] / (double)size[r] : 0.0;
  }
  free(keys);
  free(sum);
  if (rc) {
    free(nbr);
    return rc;
  }
  *nbr_out = nbr;
  *A_out = A;
  return ORC_OK;
}

/* growable u32 vector */
typedef struct {
  uint32_t *p;
  uint64_t n, cap;
} orc_vec;

static int vec_push(orc_vec *v, uint32_t x) {
  if (v->n == v->cap) {
    const uint64_t c = v->cap ? 2 * v->cap : 64;
    uint32_t *q = (uint32_t *)realloc(v->p, c * sizeof(uint32_t));
    if (!q) return ORC_NOMEM;
    v->p = q;
    v->cap = c;
  }
  v->p[v->n++] = x;
  return ORC_OK;
}

static int adj_has(const uint32_t *off, const uint32_t *nbr, uint32_t v, uint32_t u) {
  for (uint32_t s = off[v]; s < off[v + 1]; ++s)
    if (nbr[s] == u) return 1;
  return 0;
}

/* canonical_sort comparison (cliques.cpp:33-38): lexicographic over mixed lengths */
static const uint32_t *g_cl_mem;
static const uint64_t *g_cl_off;
static int cmp_clique(const void *a, const void *b) {
  const uint64_t i = *(const uint64_t *)a, j = *(const uint64_t *)b;
  const uint32_t *x = g_cl_mem + g_cl_off[i], *y = g_cl_mem + g_cl_off[j];
  const uint64_t nx = g_cl_off[i + 1] - g_cl_off[i], ny = g_cl_off[j + 1] - g_cl_off[j];
  for (uint64_t k = 0; k < nx && k < ny; ++k) {
    if (x[k] < y[k]) return -1;
    if (y[k] < x[k]) return 1;
  }
  return nx < ny ? -1 : (nx > ny ? 1 : 0);
}

/* enumerate_maximal_cliques, cliques.cpp:53-106: level k holds the k-cliques
 * (stride k); common_neighbors (:16-27) = adjacency of member 0 intersected
 * with every other member's; maximal iff empty (:91-96); children = members
 * + each common neighbor above the last member (:82-89); canonical_sort of
 * the emitted cliques (:30-49, :104). */
int orc_maximal_cliques(uint32_t R, const uint32_t *off, const uint32_t *nbr, uint32_t **c_off_out,
                        uint64_t *C_out, uint32_t **c_mem_out, uint64_t *CS_out) {
  orc_vec out_mem = {0}, out_off = {0}, front = {0}, next = {0}, common = {0};
  int rc = ORC_OK;
  *c_off_out = *c_mem_out = NULL;
  *C_out = *CS_out = 0;
  for (uint32_t v = 0; v < R && !rc; ++v) rc = vec_push(&front, v);
  rc = rc ? rc : vec_push(&out_off, 0);
  for (uint64_t k = 1; front.n && !rc; ++k) {
    const uint64_t fk = front.n / k;
    next.n = 0;
    for (uint64_t i = 0; i < fk && !rc; ++i) {
      const uint32_t *m = front.p + i * k;
      common.n = 0;
      for (uint32_t s = off[m[0]]; s < off[m[0] + 1] && !rc; ++s) {
        const uint32_t u = nbr[s];
        int all = 1;
        for (uint64_t j = 1; j < k && all; ++j) all = adj_has(off, nbr, m[j], u);
        if (all) rc = vec_push(&common, u);
      }
      for (uint64_t c = 0; c < common.n && !rc; ++c) {
        if (common.p[c] <= m[k - 1]) continue;
        for (uint64_t j = 0; j < k && !rc; ++j) rc = vec_push(&next, m[j]);
        if (!rc) rc = vec_push(&next, common.p[c]);
      }
      if (common.n == 0 && !rc) {
        for (uint64_t j = 0; j < k && !rc; ++j) rc = vec_push(&out_mem, m[j]);
        if (!rc) rc = vec_push(&out_off, (uint32_t)out_mem.n);
      }
    }
    orc_vec t = front;
    front = next;
    next = t;
  }
  free(front.p);
  free(next.p);
  free(common.p);
  if (rc) {
    free(out_mem.p);
    free(out_off.p);
    return rc;
  }
  const uint64_t C = out_off.n - 1;
  uint64_t *ord = (uint64_t *)malloc((C ? C : 1) * sizeof(uint64_t));
  uint64_t *off64 = (uint64_t *)malloc((C + 1) * sizeof(uint64_t));
  uint32_t *c_off = (uint32_t *)malloc((C + 1) * sizeof(uint32_t));
  uint32_t *c_mem = (uint32_t *)malloc((out_mem.n ? out_mem.n : 1) * sizeof(uint32_t));
  if (!ord || !off64 || !c_off || !c_mem) {
    free(ord);
    free(off64);
    free(c_off);
    free(c_mem);
    free(out_mem.p);
    free(out_off.p);
    return ORC_NOMEM;
  }
  for (uint64_t c = 0; c <= C; ++c) off64[c] = out_off.p[c];
  for (uint64_t c = 0; c < C; ++c) ord[c] = c;
  g_cl_mem = out_mem.p;
  g_cl_off = off64;
  qsort(ord, C, sizeof(uint64_t), cmp_clique);
  uint64_t pos = 0;
  c_off[0] = 0;
  for (uint64_t c = 0; c < C; ++c) {
    for (uint64_t s = off64[ord[c]]; s < off64[ord[c] + 1]; ++s) c_mem[pos++] = out_mem.p[s];
    c_off[c + 1] = (uint32_t)pos;
  }
  free(ord);
  free(off64);
  free(out_mem.p);
  free(out_off.p);
  *c_off_out = c_off;
  *c_mem_out = c_mem;
  *C_out = C;
  *CS_out = pos;
  return ORC_OK;
}
