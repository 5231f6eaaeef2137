/* TEST INFRASTRUCTURE ONLY: host restatement of the repo's synthetic-tensor
 * generator (paper_2109_09534_b200/csrc/synth.cu), so the reference arm of
 * bench.py can build the SAME tensor on the host cores and hand it to the
 * reference's own SparseTensor constructor (sparse_tensor.cpp:24-73) and
 * build_mode_views (mode_view.cpp:8-37) without loading libntcb.so.
 * tests/test_gpu_synth_host.py pins it: the canonical COO of configs 1 and
 * 2 generated here equals the device's bit for bit.
 *
 * The generator is not part of the reference (its synth_generate cannot
 * express these configs); this is an independent C
 * restatement of the same definition:
 *   candidate j:  u_{j,m} = mix(S + (j N + m + 1) G), S = fork(fork(seed, 5), 0)
 *                 uniform mode  i_m = hi32(hi32(u) * dims[m])
 *                 Zipf mode     i_m = perm_m[first k with CDF(k) > (u >> 11) 2^-53]
 *   candidates are keyed by the cell (bit-packed, or mixed radix above 64
 *   bits: both lexicographic), the first candidate of each cell is kept, and
 *   the nnz smallest kept j are the tensor (more candidates while too few);
 *   truth U_m[i, r] = (mix(fork(fork(seed, 4), m) + (i R + r + 1) G) >> 11) 2^-53;
 *   value  kind 0: max(sum_r prod_m U_m[i_m, r] + sigma g_j, 0)
 *          kind 1: rint(clip(1 + (4 model) / R + sigma g_j, 1, 5))
 *   g_j = sqrt(-2 log u1) cos(2 pi u2) from fork(fork(seed, 6), j), every
 *   operation an IEEE-rounded + - * / sqrt (log and cos by the fixed series
 *   below, no contraction: -ffp-contract=off), so host and device agree.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define G64 0x9e3779b97f4a7c15ull

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static inline uint64_t fork64(uint64_t s, uint64_t tag) { return mix64(s ^ (G64 * (tag + 1))); }

/* log(x) for x in (0, 1]: x = m 2^e, m in [sqrt(1/2), sqrt(2)),
 * log m = 2 s (1 + z/3 + z^2/5 + ... + z^11/23), s = (m-1)/(m+1), z = s^2 */
static double det_log(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  b = (b & 0xfffffffffffffull) | (1023ull << 52);
  double m;
  memcpy(&m, &b, 8);
  if (m > 1.4142135623730951) {
    m = m * 0.5;
    e += 1;
  }
  const double s = (m - 1.0) / (m + 1.0);
  const double z = s * s;
  double p = 1.0 / 23.0;
  for (int k = 10; k >= 0; --k) p = p * z + 1.0 / (double)(2 * k + 1);
  return (double)e * 0.6931471805599453 + 2.0 * s * p;
}

/* cos(2 pi u) for u in [0, 1): quadrant q = floor(4u), a = (4u - q) pi/2,
 * Taylor series of cos a / sin a to the a^22 / a^23 term */
static double det_cos2pi(double u) {
  const double t = 4.0 * u;
  const int q = (int)t;
  const double a = (t - (double)q) * 1.5707963267948966;
  const double z = a * a;
  double c = 1.0, sn = 1.0;  /* Horner from the highest term */
  for (int k = 11; k >= 1; --k) {
    c = 1.0 - z / (double)((2 * k - 1) * (2 * k)) * c;
    sn = 1.0 - z / (double)((2 * k) * (2 * k + 1)) * sn;
  }
  sn = a * sn;
  switch (q & 3) {
    case 0: return c;
    case 1: return -sn;
    case 2: return -c;
    default: return sn;
  }
}

typedef struct {
  int order;
  uint64_t d[8];
  int shift[8];
  uint64_t stride[8];
  int linear;
  const double* cdf[8];
  const uint32_t* perm[8];
} Dims;

static inline uint32_t coord_of(const Dims* d, uint64_t s_mask, uint64_t j, int m) {
  const uint64_t u = mix64(s_mask + (j * (uint64_t)d->order + (uint64_t)m + 1) * G64);
  if (!d->cdf[m]) return (uint32_t)(((u >> 32) * d->d[m]) >> 32);
  const double x = (double)(u >> 11) * 0x1.0p-53;
  const double* cdf = d->cdf[m];
  uint64_t lo = 0, hi = d->d[m] - 1;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (cdf[mid] > x)
      hi = mid;
    else
      lo = mid + 1;
  }
  return d->perm[m][lo];
}

static inline uint64_t key_of(const Dims* d, uint64_t s_mask, uint64_t j) {
  uint64_t k = 0;
  for (int m = 0; m < d->order; ++m) {
    const uint64_t c = coord_of(d, s_mask, j, m);
    if (d->linear)
      k += c * d->stride[m];
    else
      k |= c << d->shift[m];
  }
  return k;
}

/* LSD radix sort of (key, j) by the low `bits` bits of key, stable. */
static void radix_sort(uint64_t* k, uint32_t* v, uint64_t* k2, uint32_t* v2, uint64_t n, int bits,
                       int threads) {
  enum { RB = 11, NB = 1 << RB };
  const int passes = (bits + RB - 1) / RB;
  uint64_t* hist = (uint64_t*)malloc(sizeof(uint64_t) * NB * (size_t)threads);
  for (int pass = 0; pass < passes; ++pass) {
    const int sh = pass * RB;
#pragma omp parallel num_threads(threads)
    {
#ifdef _OPENMP
      const int t = omp_get_thread_num();
#else
      const int t = 0;
#endif
      const uint64_t a = n * (uint64_t)t / (uint64_t)threads, b = n * (uint64_t)(t + 1) / (uint64_t)threads;
      uint64_t* h = hist + (size_t)t * NB;
      memset(h, 0, sizeof(uint64_t) * NB);
      for (uint64_t i = a; i < b; ++i) ++h[(k[i] >> sh) & (NB - 1)];
#pragma omp barrier
#pragma omp single
      {
        uint64_t run = 0;
        for (int dg = 0; dg < NB; ++dg)
          for (int tt = 0; tt < threads; ++tt) {
            const uint64_t c = hist[(size_t)tt * NB + dg];
            hist[(size_t)tt * NB + dg] = run;
            run += c;
          }
      }
      for (uint64_t i = a; i < b; ++i) {
        const uint64_t dst = h[(k[i] >> sh) & (NB - 1)]++;
        k2[dst] = k[i];
        v2[dst] = v[i];
      }
    }
    uint64_t* tk = k; k = k2; k2 = tk;
    uint32_t* tv = v; v = v2; v2 = tv;
  }
  free(hist);
  if (passes & 1) {  /* result is in the second buffers: copy back */
    memcpy(k2, k, sizeof(uint64_t) * n);
    memcpy(v2, v, sizeof(uint32_t) * n);
  }
}

/* Returns 0, or 1 on an invalid configuration, 2 when too many candidates
 * are needed, 3 on allocation failure.  idx: nnz * order (entry-major),
 * vals: nnz.  canonical = 0: generation order (ascending candidate id, what
 * the device loads before canonicalising); 1: lexicographic order. */
int ntco_synth(int order, const uint64_t* dims, uint64_t nnz, uint64_t true_rank, double sigma,
               uint64_t seed, const double* zipf_alpha, int kind, int canonical, int threads,
               uint32_t* idx, float* vals) {
  if (order < 2 || order > 8 || (kind != 0 && kind != 1) || true_rank == 0 || true_rank > 256) return 1;
  if (threads < 1) threads = 1;
  Dims d;
  memset(&d, 0, sizeof d);
  d.order = order;
  int bits = 0;
  long double cells = 1;
  for (int m = order - 1; m >= 0; --m) {
    if (dims[m] == 0 || dims[m] > (1ull << 32)) return 1;
    d.d[m] = dims[m];
    int b = 1;
    while (b < 64 && ((dims[m] - 1) >> b)) ++b;
    d.shift[m] = bits;
    bits += b;
    cells *= (long double)dims[m];
  }
  if (bits > 64) {
    if (cells >= 18446744073709551615.0L) return 1;
    d.linear = 1;
    uint64_t st = 1;
    for (int m = order - 1; m >= 0; --m) {
      d.stride[m] = st;
      st *= dims[m];
    }
    bits = 64;
  }
  if ((long double)nnz > 0.5L * cells || nnz >= (1ull << 32)) return 1;
  const uint64_t s_mask = fork64(fork64(seed, 5), 0);
  const uint64_t noise_root = fork64(seed, 6);
  double* cdfs[8] = {0};
  uint32_t* perms[8] = {0};
  int rc = 0;
  for (int m = 0; m < order; ++m) {
    const double al = zipf_alpha ? zipf_alpha[m] : 0.0;
    if (!(al > 0.0)) continue;
    const uint64_t N = dims[m];
    double* cdf = cdfs[m] = (double*)malloc(sizeof(double) * N);
    uint32_t* perm = perms[m] = (uint32_t*)malloc(sizeof(uint32_t) * N);
    if (!cdf || !perm) { rc = 3; goto out; }
    double acc = 0.0;
    for (uint64_t k = 0; k < N; ++k) {
      acc += pow((double)(k + 1), -al);
      cdf[k] = acc;
    }
    for (uint64_t k = 0; k < N; ++k) cdf[k] /= acc;
    cdf[N - 1] = 1.0;
    for (uint64_t k = 0; k < N; ++k) perm[k] = (uint32_t)k;
    uint64_t s = fork64(fork64(seed, 7), (uint64_t)m);
    for (uint64_t k = N - 1; k > 0; --k) {  /* Fisher-Yates, Lemire next_below (rng.hpp:32-45) */
      const uint64_t bound = k + 1;
      s += G64;
      uint64_t x = mix64(s);
      unsigned __int128 mm = (unsigned __int128)x * bound;
      uint64_t lw = (uint64_t)mm;
      if (lw < bound) {
        const uint64_t th = (0 - bound) % bound;
        while (lw < th) {
          s += G64;
          x = mix64(s);
          mm = (unsigned __int128)x * bound;
          lw = (uint64_t)mm;
        }
      }
      const uint64_t r = (uint64_t)(mm >> 64);
      const uint32_t tmp = perm[k];
      perm[k] = perm[r];
      perm[r] = tmp;
    }
    d.cdf[m] = cdf;
    d.perm[m] = perm;
  }
  {
    const uint64_t kMaxCand = (1ull << 32) - 2;
    uint64_t M = nnz + (nnz / 256 > 4096 ? nnz / 256 : 4096);
    uint64_t *key = NULL, *key2 = NULL;
    uint32_t *jj = NULL, *jj2 = NULL;
    uint8_t* keep = NULL;
    uint64_t jmax = 0;
    for (;;) {
      if (M > kMaxCand) { rc = 2; goto out; }
      free(key); free(key2); free(jj); free(jj2);
      key = (uint64_t*)malloc(sizeof(uint64_t) * M);
      key2 = (uint64_t*)malloc(sizeof(uint64_t) * M);
      jj = (uint32_t*)malloc(sizeof(uint32_t) * M);
      jj2 = (uint32_t*)malloc(sizeof(uint32_t) * M);
      if (!key || !key2 || !jj || !jj2) { rc = 3; free(key); free(key2); free(jj); free(jj2); goto out; }
#pragma omp parallel for num_threads(threads) schedule(static)
      for (uint64_t j = 0; j < M; ++j) {
        key[j] = key_of(&d, s_mask, j);
        jj[j] = (uint32_t)j;
      }
      radix_sort(key, jj, key2, jj2, M, bits, threads);
      uint64_t uniq = 0;
#pragma omp parallel for num_threads(threads) reduction(+ : uniq) schedule(static)
      for (uint64_t t = 0; t < M; ++t) uniq += (t == 0 || key[t] != key[t - 1]);
      if (uniq < nnz) {
        const double frac = (double)uniq / (double)M;
        uint64_t next = (uint64_t)((double)nnz / (frac > 1e-3 ? frac : 1e-3) * 1.05) + 4096;
        if (next < M + M / 4) next = M + M / 4;
        if (next > kMaxCand && M < kMaxCand) next = kMaxCand;
        M = next;
        continue;
      }
      /* kept = first candidate of each cell; the tensor = the nnz smallest kept j */
      keep = (uint8_t*)calloc(M, 1);
      if (!keep) { rc = 3; free(key); free(key2); free(jj); free(jj2); goto out; }
#pragma omp parallel for num_threads(threads) schedule(static)
      for (uint64_t t = 0; t < M; ++t)
        if (t == 0 || key[t] != key[t - 1]) keep[jj[t]] = 1;
      uint64_t got = 0;
      for (uint64_t j = 0; j < M; ++j)
        if (keep[j] && ++got == nnz) { jmax = j; break; }
      break;
    }
    free(key2);
    free(jj2);
    /* the chosen candidate ids, in the requested order */
    uint32_t* chosen = (uint32_t*)malloc(sizeof(uint32_t) * (nnz ? nnz : 1));
    if (!chosen) { rc = 3; free(key); free(jj); free(keep); goto out; }
    uint64_t e = 0;
    if (canonical) {
      for (uint64_t t = 0; t < M && e < nnz; ++t)
        if ((t == 0 || key[t] != key[t - 1]) && jj[t] <= jmax) chosen[e++] = jj[t];
    } else {
      for (uint64_t j = 0; j <= jmax && e < nnz; ++j)
        if (keep[j]) chosen[e++] = (uint32_t)j;
    }
    free(key);
    free(jj);
    free(keep);
    /* truth factors (factor_set.cpp:18-27 layout) and the values */
    const int R = (int)true_rank;
    double* truth[8] = {0};
    for (int m = 0; m < order; ++m) {
      const uint64_t n = dims[m] * (uint64_t)R;
      truth[m] = (double*)malloc(sizeof(double) * n);
      if (!truth[m]) { rc = 3; break; }
      const uint64_t root = fork64(fork64(seed, 4), (uint64_t)m);
#pragma omp parallel for num_threads(threads) schedule(static)
      for (uint64_t q = 0; q < n; ++q) truth[m][q] = (double)(mix64(root + (q + 1) * G64) >> 11) * 0x1.0p-53;
    }
    if (rc == 0) {
#pragma omp parallel for num_threads(threads) schedule(static)
      for (uint64_t t = 0; t < nnz; ++t) {
        const uint64_t j = chosen[t];
        uint32_t ix[8];
        for (int m = 0; m < order; ++m) {
          ix[m] = coord_of(&d, s_mask, j, m);
          idx[t * (uint64_t)order + (uint64_t)m] = ix[m];
        }
        double model = 0.0;
        for (int r = 0; r < R; ++r) {
          double prod = 1.0;
          for (int m = 0; m < order; ++m) prod = prod * truth[m][(uint64_t)ix[m] * (uint64_t)R + (uint64_t)r];
          model = model + prod;
        }
        double g = 0.0;
        if (sigma > 0.0) {
          uint64_t s = fork64(noise_root, j);
          s += G64;
          const double u1 = (double)((mix64(s) >> 11) + 1) * 0x1.0p-53;
          s += G64;
          const double u2 = (double)(mix64(s) >> 11) * 0x1.0p-53;
          g = sqrt(-2.0 * det_log(u1)) * det_cos2pi(u2);
        }
        double v;
        if (kind == 1) {
          v = (1.0 + (4.0 * model) / (double)R) + sigma * g;
          v = rint(fmin(fmax(v, 1.0), 5.0));
        } else {
          v = model + sigma * g;
          v = v > 0.0 ? v : 0.0;
        }
        vals[t] = (float)v;
      }
    }
    for (int m = 0; m < order; ++m) free(truth[m]);
    free(chosen);
  }
out:
  for (int m = 0; m < 8; ++m) {
    free(cdfs[m]);
    free(perms[m]);
  }
  return rc;
}
