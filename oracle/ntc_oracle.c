/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into, called by, or
 * shipped with the product library (paper_2109_09534_b200/libntcb.so).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * A plain-C restatement of the reference's hot path (arXiv 2109.09534,
 * "ntc" library under /root/reference/proj/core), in fp64 exactly as the
 * reference evaluates it, operation for operation, so that on x86-64 without
 * FMA contraction its results are BIT-IDENTICAL to the reference's (pinned by
 * tests/test_oracle.py against the compiled reference oracle/_ref and the
 * golden vectors in tests/golden/).
 *
 * Each function cites the reference file:line it restates.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_G 0x9e3779b97f4a7c15ull

/* Error codes mirror the reference exception classes:
 * 1 invalid_argument, 2 runtime_error, 3 out_of_range, 4 domain_error. */
static __thread char g_err[256];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ---- RngStream: proj/core/include/ntc/rng.hpp:13-63 --------------------- */
uint64_t orc_mix(uint64_t z) { /* rng.hpp:55-59 */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
uint64_t orc_fork(uint64_t state, uint64_t tag) { /* rng.hpp:18-20 */
  return orc_mix(state ^ (ORC_G * (tag + 1)));
}
static inline uint64_t next_u64(uint64_t* s) { /* rng.hpp:22-25 */
  *s += ORC_G;
  return orc_mix(*s);
}
static inline double next_double(uint64_t* s) { /* rng.hpp:28 */
  return (double)(next_u64(s) >> 11) * 0x1.0p-53;
}
static inline uint64_t next_below(uint64_t* s, uint64_t bound) { /* rng.hpp:32-45 */
  uint64_t x = next_u64(s);
  unsigned __int128 m = (unsigned __int128)x * bound;
  uint64_t lo = (uint64_t)m;
  if (lo < bound) {
    const uint64_t threshold = (0 - bound) % bound;
    while (lo < threshold) {
      x = next_u64(s);
      m = (unsigned __int128)x * bound;
      lo = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}

void orc_next_u64_n(uint64_t state, int n, uint64_t* out) {
  for (int i = 0; i < n; ++i) out[i] = next_u64(&state);
}
void orc_next_double_n(uint64_t state, int n, double* out) {
  for (int i = 0; i < n; ++i) out[i] = next_double(&state);
}
void orc_next_below_n(uint64_t state, uint64_t bound, int n, uint64_t* out) {
  for (int i = 0; i < n; ++i) out[i] = next_below(&state, bound);
}

/* sweep_stream(seed, k, mode) raw state: ao.cpp:16-17 (kTagSweep = 2), 65-68 */
uint64_t orc_sweep_state(uint64_t seed, uint64_t sweep, int mode) {
  return orc_fork(orc_fork(orc_fork(seed, 2), sweep), (uint64_t)mode);
}

/* ---- sampling: nmc.cpp:36-63 -------------------------------------------- */
uint64_t orc_blocksize(double c, uint64_t n) { /* nmc.cpp:36-40 */
  if (c >= 1.0) return n;
  const uint64_t b = (uint64_t)floor(c * (double)n);
  return b > n ? n : b;
}

/* Partial Fisher-Yates (nmc.cpp:44-63).  perm: scratch of n uint32. */
static uint64_t sample_into(uint64_t n, double c, uint64_t state, uint32_t* picks,
                            uint32_t* perm) {
  const uint64_t b = orc_blocksize(c, n);
  if (b == 0) return 0;
  if (c >= 1.0) {
    for (uint64_t t = 0; t < n; ++t) picks[t] = (uint32_t)t;
    return b;
  }
  for (uint64_t t = 0; t < n; ++t) perm[t] = (uint32_t)t;
  for (uint64_t j = 0; j < b; ++j) {
    const uint64_t r = j + next_below(&state, n - j);
    const uint32_t tmp = perm[j];
    perm[j] = perm[r];
    perm[r] = tmp;
    picks[j] = perm[j];
  }
  return b;
}

uint64_t orc_sample_row(uint64_t n, double c, uint64_t state, uint32_t* picks) {
  uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  const uint64_t b = sample_into(n, c, state, picks, perm);
  free(perm);
  return b;
}

/* Sampled set of every row of a view, sample_row with the row stream
 * fork(root, p) (nmc.cpp:236): out[e] = 1 for the picked entries of each
 * slice (absolute view positions, rows in parallel). */
void orc_sample_mask_rows(uint64_t rows, const uint64_t* off, double c, uint64_t root, uint8_t* out,
                          int threads) {
#pragma omp parallel num_threads(threads)
  {
    uint64_t cap = 0;
    uint32_t *picks = NULL, *perm = NULL;
#pragma omp for schedule(dynamic, 16)
    for (uint64_t p = 0; p < rows; ++p) {
      const uint64_t n = off[p + 1] - off[p];
      if (n > cap) {
        free(picks);
        free(perm);
        cap = n;
        picks = (uint32_t*)malloc(sizeof(uint32_t) * cap);
        perm = (uint32_t*)malloc(sizeof(uint32_t) * cap);
      }
      memset(out + off[p], 0, n);
      const uint64_t b = sample_into(n, c, orc_fork(root, p), picks, perm);
      for (uint64_t j = 0; j < b; ++j) out[off[p] + picks[j]] = 1;
    }
    free(picks);
    free(perm);
  }
}

/* ---- SparseTensor canonicalisation: sparse_tensor.cpp:24-73 -------------- */
typedef struct {
  const uint32_t* idx;
  int order;
} lex_ctx;

static int lex_cmp(const void* a, const void* b, void* arg) {
  const lex_ctx* c = (const lex_ctx*)arg;
  const uint32_t* ka = c->idx + (*(const uint64_t*)a) * (uint64_t)c->order;
  const uint32_t* kb = c->idx + (*(const uint64_t*)b) * (uint64_t)c->order;
  for (int m = 0; m < c->order; ++m) {
    if (ka[m] < kb[m]) return -1;
    if (ka[m] > kb[m]) return 1;
  }
  return 0;
}

int orc_canonicalize(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* idx,
                     const double* vals, uint32_t* out_idx, double* out_vals) {
  if (order < 2) return fail(1, "SparseTensor: order must be >= 2");
  for (int m = 0; m < order; ++m)
    if (dims[m] == 0) return fail(1, "SparseTensor: dimensions must be positive");
  for (uint64_t e = 0; e < nnz; ++e) {
    for (int m = 0; m < order; ++m)
      if (idx[e * order + m] >= dims[m]) {
        snprintf(g_err, sizeof g_err, "SparseTensor: index out of bounds at entry %llu",
                 (unsigned long long)e);
        return 1;
      }
    const double v = vals[e];
    if (!isfinite(v)) {
      snprintf(g_err, sizeof g_err, "SparseTensor: non-finite value at entry %llu",
               (unsigned long long)e);
      return 1;
    }
    if (v < 0.0) {
      snprintf(g_err, sizeof g_err, "SparseTensor: negative value at entry %llu",
               (unsigned long long)e);
      return 1;
    }
  }
  uint64_t* perm = (uint64_t*)malloc(sizeof(uint64_t) * (nnz ? nnz : 1));
  for (uint64_t e = 0; e < nnz; ++e) perm[e] = e;
  lex_ctx ctx = {idx, order};
  qsort_r(perm, nnz, sizeof(uint64_t), lex_cmp, &ctx);
  for (uint64_t e = 0; e < nnz; ++e) {
    memcpy(out_idx + e * order, idx + perm[e] * order, sizeof(uint32_t) * order);
    out_vals[e] = vals[perm[e]];
  }
  free(perm);
  for (uint64_t e = 1; e < nnz; ++e) {
    if (memcmp(out_idx + (e - 1) * order, out_idx + e * order, sizeof(uint32_t) * order) == 0) {
      int n = snprintf(g_err, sizeof g_err, "SparseTensor: duplicate index (");
      for (int m = 0; m < order && n < (int)sizeof g_err; ++m)
        n += snprintf(g_err + n, sizeof g_err - n, "%s%u", m ? "," : "",
                      out_idx[e * order + m] + 1);
      if (n < (int)sizeof g_err) snprintf(g_err + n, sizeof g_err - n, ")");
      return 1;
    }
  }
  return 0;
}

/* ---- build_mode_views: mode_view.cpp:8-37 (stable counting sort) -------- */
void orc_build_view(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* idx,
                    const double* vals, int mode, uint64_t* offsets, uint32_t* others,
                    double* values) {
  const uint64_t rows = dims[mode];
  memset(offsets, 0, sizeof(uint64_t) * (rows + 1));
  for (uint64_t e = 0; e < nnz; ++e) ++offsets[idx[e * order + mode] + 1];
  for (uint64_t p = 1; p <= rows; ++p) offsets[p] += offsets[p - 1];
  uint64_t* cursor = (uint64_t*)malloc(sizeof(uint64_t) * (rows ? rows : 1));
  memcpy(cursor, offsets, sizeof(uint64_t) * rows);
  for (uint64_t e = 0; e < nnz; ++e) {
    const uint32_t* ix = idx + e * order;
    const uint64_t t = cursor[ix[mode]]++;
    values[t] = vals[e];
    uint32_t* dst = others + t * (order - 1);
    for (int q = 0; q < order; ++q)
      if (q != mode) *dst++ = ix[q];
  }
  free(cursor);
}

/* ---- per-row numerics: nmc.cpp:68-106, 140-197, factor_set.cpp:42-64 ---- */
typedef struct {
  int order;
  int mode;
  uint64_t rank;
  const uint64_t* dims;
  const double* const* factors; /* factors[m]: dims[m] x rank, row-major */
} kr_ctx;

static void kr_row(const kr_ctx* k, const uint32_t* oth, double* out) { /* factor_set.cpp:42-64 */
  int first = 1, pos = 0;
  for (int m = 0; m < k->order; ++m) {
    if (m == k->mode) continue;
    const double* row = k->factors[m] + (uint64_t)oth[pos++] * k->rank;
    if (first) {
      for (uint64_t r = 0; r < k->rank; ++r) out[r] = row[r];
      first = 0;
    } else {
      for (uint64_t r = 0; r < k->rank; ++r) out[r] *= row[r];
    }
  }
}

/* accumulate_row (nmc.cpp:68-106): gradient at y and Hessian (full, mirrored). */
static void accumulate_row(const kr_ctx* k, const uint32_t* others, const double* values,
                           uint64_t base, const uint32_t* picks, uint64_t b,
                           const double* y, double lambda, double* w, double* z, double* grad,
                           double* h, double* kr) {
  const uint64_t R = k->rank;
  const int no = k->order - 1;
  for (uint64_t r = 0; r < R; ++r) w[r] = z[r] = 0.0;
  for (uint64_t r = 0; r < R; ++r)
    for (uint64_t q = 0; q < R; ++q) h[r * R + q] = (r == q) ? lambda : 0.0;
  for (uint64_t j = 0; j < b; ++j) {
    const uint64_t t = base + picks[j];
    kr_row(k, others + t * no, kr);
    const double x = values[t];
    double dot = 0.0;
    for (uint64_t r = 0; r < R; ++r) dot += y[r] * kr[r];
    for (uint64_t r = 0; r < R; ++r) w[r] -= x * kr[r];
    for (uint64_t r = 0; r < R; ++r) z[r] += dot * kr[r];
    for (uint64_t r = 0; r < R; ++r)
      for (uint64_t q = r; q < R; ++q) h[r * R + q] += kr[r] * kr[q];
  }
  for (uint64_t r = 0; r < R; ++r)
    for (uint64_t q = 0; q < r; ++q) h[r * R + q] = h[q * R + r];
  for (uint64_t r = 0; r < R; ++r) grad[r] = w[r] + z[r] + lambda * y[r];
}

/* power_method (nmc.cpp:140-172).  Returns 0 ok, 1 invalid_argument. */
int orc_power_method(uint64_t n, const double* h, int max_iters, double tol, double* out) {
  if (n == 0) return fail(1, "power_method: square matrix required");
  if (max_iters < 1) return fail(1, "power_method: max_iters must be >= 1");
  for (uint64_t i = 0; i < n * n; ++i)
    if (!isfinite(h[i])) return fail(1, "power_method: non-finite entries in matrix");
  double v[64], u[64];
  double* vv = n <= 64 ? v : (double*)malloc(sizeof(double) * n);
  double* uu = n <= 64 ? u : (double*)malloc(sizeof(double) * n);
  for (uint64_t i = 0; i < n; ++i) vv[i] = 1.0 / sqrt((double)n);
  double rq = 0.0, rq_prev = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    for (uint64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (uint64_t j = 0; j < n; ++j) s += h[i * n + j] * vv[j];
      uu[i] = s;
    }
    double num = 0.0, unorm2 = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
      num += vv[i] * uu[i];
      unorm2 += uu[i] * uu[i];
    }
    rq = num;
    if (unorm2 == 0.0) {
      rq = 0.0;
      break;
    }
    if (it > 0 && fabs(rq - rq_prev) <= tol * fabs(rq)) break;
    rq_prev = rq;
    const double inv = 1.0 / sqrt(unorm2);
    for (uint64_t i = 0; i < n; ++i) vv[i] = uu[i] * inv;
  }
  if (vv != v) free(vv);
  if (uu != u) free(uu);
  *out = rq;
  return 0;
}

/* row_step (nmc.cpp:174-197). */
int orc_row_step(uint64_t rank, const double* y, const double* a_prev, const double* grad,
                 double lipschitz, double lambda, double* a_new, double* y_new, double* beta) {
  if (!(lambda > 0.0)) return fail(1, "row_step: lambda must be > 0");
  if (!(lipschitz >= lambda)) return fail(1, "row_step: step constant below lambda");
  const double inv_l = 1.0 / lipschitz;
  const double sl = sqrt(lipschitz), sm = sqrt(lambda);
  const double bt = (sl - sm) / (sl + sm);
  for (uint64_t r = 0; r < rank; ++r) {
    const double a = y[r] - inv_l * grad[r];
    a_new[r] = a > 0.0 ? a : 0.0;
  }
  for (uint64_t r = 0; r < rank; ++r) y_new[r] = a_new[r] + bt * (a_new[r] - a_prev[r]);
  if (beta) *beta = bt;
  return 0;
}

/* Gradient / Hessian of one row for an explicit pick list (row_gradient /
 * row_hessian, nmc.cpp:120-138). */
void orc_row_terms(int order, const uint64_t* dims, uint64_t rank, const double* const* factors,
                   int mode, const uint64_t* offsets, const uint32_t* others,
                   const double* values, uint64_t row, const uint32_t* picks, uint64_t b,
                   const double* y, double lambda, double* w, double* z, double* grad,
                   double* h) {
  kr_ctx k = {order, mode, rank, dims, factors};
  double* kr = (double*)malloc(sizeof(double) * rank);
  accumulate_row(&k, others, values, offsets[row], picks, b, y, lambda, w, z, grad, h, kr);
  free(kr);
}

typedef struct {
  double lambda;
  double c;
  int max_inner;
  int power_iters;
  double power_tol;
  int threads;
  int chunk;
} orc_nmc_cfg;

/* NmcConfig::validate (nmc.cpp:13-23). */
int orc_nmc_validate(const orc_nmc_cfg* c) {
  if (!(c->lambda > 0.0)) return fail(1, "NmcConfig: lambda must be > 0");
  if (!(c->c > 0.0 && c->c <= 1.0)) return fail(1, "NmcConfig: c must be in (0, 1]");
  if (c->max_inner < 0) return fail(1, "NmcConfig: max_inner must be >= 0");
  if (c->power_iters < 1) return fail(1, "NmcConfig: power_iters must be >= 1");
  if (!(c->power_tol > 0.0)) return fail(1, "NmcConfig: power_tol must be > 0");
  if (c->threads < 1) return fail(1, "NmcConfig: threads must be >= 1");
  if (c->chunk < 0) return fail(1, "NmcConfig: chunk must be >= 0");
  return 0;
}

/*
 * s_nmc (nmc.cpp:199-272) restricted to rows [row_begin, row_end) of view
 * `mode` (the full range reproduces the reference call; a sub-range is the
 * per-rank shard of the multi-GPU partition, which is valid because rows are
 * independent and every row's stream is fork(l).fork(p) of `rng_state`).
 * factors[mode]/momentum[mode] are overwritten on the row range: A = Y =
 * a_init (momentum reset, nmc.cpp:212-215), then max_inner inner iterations.
 * a_init may alias factors[mode] (ao.cpp:123).
 */
int orc_s_nmc(int order, const uint64_t* dims, uint64_t rank, double* const* factors,
              double* const* momentum, int mode, const uint64_t* offsets,
              const uint32_t* others, const double* values, const double* a_init,
              const orc_nmc_cfg* cfg, uint64_t rng_state, uint64_t row_begin,
              uint64_t row_end, uint64_t* accessed_out) {
  int rc = orc_nmc_validate(cfg);
  if (rc) return rc;
  if (mode < 0 || mode >= order) return fail(1, "s_nmc: mode out of range");
  const uint64_t R = rank;
  double* A = factors[mode];
  double* Y = momentum[mode];
  for (uint64_t i = row_begin * R; i < row_end * R; ++i)
    if (!(a_init[i] >= 0.0)) return fail(1, "s_nmc: a_init must be nonnegative");
  if (A != a_init) memmove(A + row_begin * R, a_init + row_begin * R, sizeof(double) * (row_end - row_begin) * R);
  memcpy(Y + row_begin * R, A + row_begin * R, sizeof(double) * (row_end - row_begin) * R);

  kr_ctx k = {order, mode, R, dims, (const double* const*)factors};
  uint64_t accessed = 0;
  int failed = 0;
  int fail_code = 0;
  char diag[256] = {0};
  uint64_t max_n = 0;
  for (uint64_t p = row_begin; p < row_end; ++p) {
    const uint64_t n = offsets[p + 1] - offsets[p];
    if (n > max_n) max_n = n;
  }

#pragma omp parallel num_threads(cfg->threads) reduction(+ : accessed)
  {
    double* ws = (double*)malloc(sizeof(double) * (7 * R + R * R));
    double *w = ws, *z = ws + R, *grad = ws + 2 * R, *kr = ws + 3 * R, *aprev = ws + 4 * R,
           *h = ws + 5 * R;
    uint32_t* picks = (uint32_t*)malloc(sizeof(uint32_t) * (max_n ? max_n : 1));
    uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * (max_n ? max_n : 1));
    for (int l = 0; l < cfg->max_inner; ++l) {
#pragma omp for schedule(static)
      for (int64_t pi = (int64_t)row_begin; pi < (int64_t)row_end; ++pi) {
        int f;
#pragma omp atomic read
        f = failed;
        if (f) continue;
        const uint64_t p = (uint64_t)pi;
        const uint64_t n = offsets[p + 1] - offsets[p];
        const uint64_t st = orc_fork(orc_fork(rng_state, (uint64_t)l), p);
        const uint64_t b = sample_into(n, cfg->c, st, picks, perm);
        if (b == 0) continue;
        accessed += b;
        double* y = Y + p * R;
        double* a = A + p * R;
        memcpy(aprev, a, sizeof(double) * R);
        accumulate_row(&k, others, values, offsets[p], picks, b, y, cfg->lambda, w, z, grad, h,
                       kr);
        char msg[256];
        int code = 0;
        for (uint64_t r = 0; r < R; ++r)
          if (!isfinite(grad[r])) {
            snprintf(msg, sizeof msg, "s_nmc: non-finite gradient at row %llu (mode %d)",
                     (unsigned long long)(p + 1), mode + 1);
            code = 2;
            break;
          }
        double est = 0.0;
        if (!code && orc_power_method(R, h, cfg->power_iters, cfg->power_tol, &est)) {
          snprintf(msg, sizeof msg, "%s", g_err);
          code = 2;
        }
        if (!code) {
          const double lip = est * 1.01;
          if (orc_row_step(R, y, aprev, grad, lip, cfg->lambda, a, y, NULL)) {
            snprintf(msg, sizeof msg, "%s", g_err);
            code = 2;
          }
        }
        if (code) {
#pragma omp critical(orc_diag)
          {
            if (!failed) {
              failed = 1;
              fail_code = code;
              snprintf(diag, sizeof diag, "%s", msg);
            }
          }
        }
      }
    }
    free(ws);
    free(picks);
    free(perm);
  }
  if (failed) return fail(fail_code, diag);
  if (accessed_out) *accessed_out += accessed;
  return 0;
}

/* ---- metrics: metrics.cpp:8-37, factor_set.cpp:72-86 --------------------- */
static double cpd_value(int order, uint64_t rank, const double* const* factors,
                        const uint32_t* ix) {
  double total = 0.0;
  for (uint64_t r = 0; r < rank; ++r) {
    double prod = 1.0;
    for (int m = 0; m < order; ++m) prod *= factors[m][(uint64_t)ix[m] * rank + r];
    total += prod;
  }
  return total;
}

/* Serial SSE / sum x^2 / sum ||U||^2 in canonical entry order. */
void orc_metrics(int order, const uint64_t* dims, uint64_t rank, const double* const* factors,
                 uint64_t nnz, const uint32_t* idx, const double* vals, double* sse,
                 double* sumsq, double* reg) {
  double fit = 0.0, den = 0.0;
  for (uint64_t e = 0; e < nnz; ++e) {
    const double x = vals[e];
    const double d = x - cpd_value(order, rank, factors, idx + e * order);
    fit += d * d;
    den += x * x;
  }
  double rg = 0.0;
  for (int m = 0; m < order; ++m) {
    double s = 0.0; /* Matrix::frob_norm_sq, matrix.hpp:33-37 */
    for (uint64_t i = 0; i < dims[m] * rank; ++i) s += factors[m][i] * factors[m][i];
    rg += s;
  }
  *sse = fit;
  *sumsq = den;
  *reg = rg;
}

/* objective = 0.5*SSE + 0.5*lambda*sum||U||^2 (metrics.cpp:8-21). */
int orc_objective(int order, const uint64_t* dims, uint64_t rank, const double* const* factors,
                  uint64_t nnz, const uint32_t* idx, const double* vals, double lambda,
                  double* out) {
  if (lambda < 0.0) return fail(1, "objective: lambda must be >= 0");
  double sse, den, reg;
  orc_metrics(order, dims, rank, factors, nnz, idx, vals, &sse, &den, &reg);
  *out = 0.5 * sse + 0.5 * lambda * reg;
  return 0;
}

/* relative_error = sqrt(SSE)/sqrt(sum x^2) (metrics.cpp:23-37). */
int orc_relative_error(int order, const uint64_t* dims, uint64_t rank,
                       const double* const* factors, uint64_t nnz, const uint32_t* idx,
                       const double* vals, double* out) {
  double sse, den, reg;
  orc_metrics(order, dims, rank, factors, nnz, idx, vals, &sse, &den, &reg);
  if (den == 0.0) return fail(4, "relative_error: all observed values are zero");
  *out = sqrt(sse) / sqrt(den);
  return 0;
}

/* initial_factors (ao.cpp:70-73 -> factor_set.cpp:18-27): mode m filled
 * row-major from RngStream(seed).fork(1).fork(m).next_double(). */
void orc_initial_factors(int order, const uint64_t* dims, uint64_t rank, uint64_t seed,
                         double* out) {
  const uint64_t base = orc_fork(seed, 1);
  uint64_t pos = 0;
  for (int m = 0; m < order; ++m) {
    uint64_t s = orc_fork(base, (uint64_t)m);
    for (uint64_t i = 0; i < dims[m] * rank; ++i) out[pos++] = next_double(&s);
  }
}
