// Synthetic tensors of the BASELINE.json shapes, generated on the device.
// (Not part of the reference: its synth_generate (synth.cpp:84-145) cannot
// express exact-count sampling, Zipf modes or these sizes.)
//
// Candidate cell j has coordinates drawn from u_{j,m} = mix(S_mask + (j*N + m
// + 1) G), S_mask = fork(fork(seed, 5), 0):
//   uniform mode:  i_m = hi32( hi32(u) * dims[m] )
//   Zipf(alpha):   rank k = first k with CDF(k) > (u >> 11) 2^-53 over
//                  P(k) ~ (k+1)^-alpha, then i_m = perm_m[k] with perm_m a
//                  seeded Fisher-Yates permutation of the ids (stream
//                  fork(fork(seed, 7), m)) -- "Zipf over randomly permuted ids".
// Candidates are taken in j order and a cell already seen is redrawn
// (= skipped) until nnz unique cells exist.  Truth factors U_m[i, r] =
// next_double of fork(fork(seed, 4), m) at index i*R + r (row-major, as
// FactorSet::random_uniform, factor_set.cpp:18-27).  Values:
//   kind 0: sum_r prod_m U_m[i_m, r] + sigma g_j, clamped at 0;
//   kind 1: round(clip(1 + 4 * (sum_r prod_m U_m[i_m, r]) / R_true + sigma g_j, 1, 5))
//           (the 1-5 rating model of BASELINE configs[2]);
// g_j is the reference's Box-Muller (rng.hpp:49-53) on fork(fork(seed, 6), j),
// with log and cos evaluated by fixed series (det_log, det_cos2pi) and every
// floating-point operation an explicitly rounded + - * / sqrt (no FMA
// contraction): the values are reproducible bit for bit on the host, which
// the reference arm of bench.py relies on (oracle/synth_host.c, pinned by
// tests/test_gpu_synth_host.py).  Tags 4..6 follow synth.cpp:16-18.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace ntcb {

void load_tensor_f32(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                     const uint32_t* idx, const float* vals, bool on_device);

namespace {

template <class T>
struct Buf {
  T* p = nullptr;
  explicit Buf(size_t n) {
    if (n) NTCB_CUDA(cudaMalloc(&p, sizeof(T) * n));
  }
  ~Buf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
  }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
};

struct Dims {
  uint64_t d[NTCB_MAX_ORDER];
  int shift[NTCB_MAX_ORDER];
  uint64_t stride[NTCB_MAX_ORDER];  // mixed-radix linear key when the bit-packed one exceeds 64 bits
  int linear;
  const double* cdf[NTCB_MAX_ORDER];     // Zipf modes: CDF over ranks (nullptr = uniform)
  const uint32_t* perm[NTCB_MAX_ORDER];  // Zipf modes: rank -> id
  int order;
};

__device__ __forceinline__ uint32_t coord_of(const Dims& d, uint64_t s_mask, uint64_t j, int m) {
  const uint64_t u = mix64(s_mask + (j * d.order + m + 1) * kGolden);
  if (d.cdf[m] == nullptr) return static_cast<uint32_t>(((u >> 32) * d.d[m]) >> 32);
  const double x = static_cast<double>(u >> 11) * 0x1.0p-53;
  const double* cdf = d.cdf[m];
  uint64_t lo = 0, hi = d.d[m] - 1;  // first k with cdf[k] > x (cdf[last] == 1)
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (cdf[mid] > x)
      hi = mid;
    else
      lo = mid + 1;
  }
  return d.perm[m][lo];
}

__global__ void k_candidates(uint64_t s_mask, uint64_t M, Dims d, uint64_t* key, uint32_t* jj) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < M;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t k = 0;
    if (d.linear)
      for (int m = 0; m < d.order; ++m) k += static_cast<uint64_t>(coord_of(d, s_mask, j, m)) * d.stride[m];
    else
      for (int m = 0; m < d.order; ++m) k |= static_cast<uint64_t>(coord_of(d, s_mask, j, m)) << d.shift[m];
    key[j] = k;
    jj[j] = static_cast<uint32_t>(j);
  }
}

// first occurrence of each cell (the sort is stable, so j ascends in a run)
__global__ void k_first(const uint64_t* skey, const uint32_t* sj, uint64_t M, uint32_t* keep_j,
                        unsigned long long* count) {
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < M;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const bool first = t == 0 || skey[t] != skey[t - 1];
    keep_j[t] = first ? sj[t] : 0xffffffffu;
    if (first) atomicAdd(count, 1ull);
  }
}

__global__ void k_truth(uint64_t root, uint64_t n, double* out) {
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[q] = static_cast<double>(mix64(root + (q + 1) * kGolden) >> 11) * 0x1.0p-53;
}

// log(x), x in (0, 1]: x = m 2^e with m in [sqrt(1/2), sqrt(2)),
// log m = 2 s (1 + z/3 + ... + z^11/23), s = (m - 1)/(m + 1), z = s^2
__device__ double det_log(double x) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  int e = static_cast<int>((b >> 52) & 0x7ff) - 1023;
  b = (b & 0xfffffffffffffull) | (1023ull << 52);
  double m = __longlong_as_double(static_cast<long long>(b));
  if (m > 1.4142135623730951) {
    m = __dmul_rn(m, 0.5);
    e += 1;
  }
  const double s = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
  const double z = __dmul_rn(s, s);
  double p = __ddiv_rn(1.0, 23.0);
  for (int k = 10; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, z), __ddiv_rn(1.0, static_cast<double>(2 * k + 1)));
  return __dadd_rn(__dmul_rn(static_cast<double>(e), 0.6931471805599453), __dmul_rn(__dmul_rn(2.0, s), p));
}

// cos(2 pi u), u in [0, 1): quadrant q = floor(4u), a = (4u - q) pi/2,
// Taylor series of cos a and sin a to the a^22 / a^23 term (Horner)
__device__ double det_cos2pi(double u) {
  const double t = __dmul_rn(4.0, u);
  const int q = static_cast<int>(t);
  const double a = __dmul_rn(__dsub_rn(t, static_cast<double>(q)), 1.5707963267948966);
  const double z = __dmul_rn(a, a);
  double c = 1.0, sn = 1.0;
  for (int k = 11; k >= 1; --k) {
    c = __dsub_rn(1.0, __dmul_rn(__ddiv_rn(z, static_cast<double>((2 * k - 1) * (2 * k))), c));
    sn = __dsub_rn(1.0, __dmul_rn(__ddiv_rn(z, static_cast<double>((2 * k) * (2 * k + 1))), sn));
  }
  sn = __dmul_rn(a, sn);
  switch (q & 3) {
    case 0: return c;
    case 1: return -sn;
    case 2: return -c;
    default: return sn;
  }
}

__global__ void k_emit(const uint32_t* js, uint64_t nnz, uint64_t s_mask, Dims d, int R,
                       const double* const* truth, uint64_t noise_root, double sigma, int kind,
                       uint32_t* idx, float* vals) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t j = js[e];
    uint32_t ix[NTCB_MAX_ORDER];
    for (int m = 0; m < d.order; ++m) {
      ix[m] = coord_of(d, s_mask, j, m);
      idx[e * d.order + m] = ix[m];
    }
    double model = 0.0;
    for (int r = 0; r < R; ++r) {
      double prod = 1.0;
      for (int m = 0; m < d.order; ++m) prod = __dmul_rn(prod, truth[m][static_cast<uint64_t>(ix[m]) * R + r]);
      model = __dadd_rn(model, prod);
    }
    double g = 0.0;
    if (sigma > 0.0) {
      uint64_t s = fork64(noise_root, j);
      s += kGolden;
      const double u1 = static_cast<double>((mix64(s) >> 11) + 1) * 0x1.0p-53;
      s += kGolden;
      const double u2 = static_cast<double>(mix64(s) >> 11) * 0x1.0p-53;
      g = __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, det_log(u1))), det_cos2pi(u2));
    }
    double v;
    if (kind == 1) {
      v = __dadd_rn(__dadd_rn(1.0, __ddiv_rn(__dmul_rn(4.0, model), static_cast<double>(R))), __dmul_rn(sigma, g));
      v = rint(fmin(fmax(v, 1.0), 5.0));
    } else {
      v = __dadd_rn(model, __dmul_rn(sigma, g));
      v = v > 0.0 ? v : 0.0;
    }
    vals[e] = static_cast<float>(v);
  }
}

unsigned grid_of(uint64_t n, int sms) {
  uint64_t g = (n + 255) / 256;
  const uint64_t cap = static_cast<uint64_t>(sms) * 16;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min(g, cap)));
}

// host splitmix64 stream (rng.hpp semantics)
struct HostRng {
  uint64_t s;
  uint64_t next() {
    s += kGolden;
    return mix64(s);
  }
  uint64_t below(uint64_t bound) {  // Lemire with rejection (rng.hpp:32-45)
    uint64_t x = next();
    unsigned __int128 m = static_cast<unsigned __int128>(x) * bound;
    uint64_t lo = static_cast<uint64_t>(m);
    if (lo < bound) {
      const uint64_t th = (0 - bound) % bound;
      while (lo < th) {
        x = next();
        m = static_cast<unsigned __int128>(x) * bound;
        lo = static_cast<uint64_t>(m);
      }
    }
    return static_cast<uint64_t>(m >> 64);
  }
};

}  // namespace

void synth_general(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                   uint64_t true_rank, double sigma, uint64_t seed, const double* zipf_alpha,
                   int kind) {
  if (order < 2 || order > NTCB_MAX_ORDER) fail(NTCB_EINVAL, "synth: order must be in [2, 8]");
  if (kind != 0 && kind != 1) fail(NTCB_EINVAL, "synth: unknown value kind");
  Dims d{};
  d.order = order;
  int bits = 0;
  long double cells = 1;
  for (int m = order - 1; m >= 0; --m) {
    if (dims[m] == 0 || dims[m] > (1ull << 32)) fail(NTCB_EINVAL, "synth: bad dimension");
    d.d[m] = dims[m];
    int b = 1;
    while (b < 64 && (dims[m] - 1) >> b) ++b;
    d.shift[m] = bits;
    bits += b;
    cells *= static_cast<long double>(dims[m]);
  }
  if (bits > 64) {
    // the cell id as a mixed-radix number (4.8M x 1.8M x 1.8M = 1.6e19 < 2^64)
    if (cells >= 18446744073709551615.0L) fail(NTCB_EINVAL, "synth: cell space exceeds 2^64");
    d.linear = 1;
    uint64_t st = 1;
    for (int m = order - 1; m >= 0; --m) {
      d.stride[m] = st;
      st *= dims[m];
    }
    bits = 64;
  }
  if (static_cast<long double>(nnz) > 0.5L * cells)
    fail(NTCB_EINVAL, "synth: nnz exceeds half the cell space");
  if (true_rank == 0 || true_rank > 256) fail(NTCB_EINVAL, "synth: bad true rank");
  if (nnz >= (1ull << 32)) fail(NTCB_EINVAL, "synth: nnz must be < 2^32 per device");
  cudaStream_t st = ctx->stream;
  const int sms = ctx->sm_count;
  const uint64_t s_mask = fork64(fork64(seed, 5), 0);
  const uint64_t noise_root = fork64(seed, 6);

  // Zipf tables: CDF over ranks and a seeded id permutation per Zipf mode
  std::vector<double*> d_cdf(order, nullptr);
  std::vector<uint32_t*> d_perm(order, nullptr);
  struct Cleanup {
    std::vector<double*>& a;
    std::vector<uint32_t*>& b;
    ~Cleanup() {
      for (auto* p : a)
        if (p) cudaFree(p);
      for (auto* p : b)
        if (p) cudaFree(p);
    }
  } cleanup{d_cdf, d_perm};
  for (int m = 0; m < order; ++m) {
    const double al = zipf_alpha ? zipf_alpha[m] : 0.0;
    if (!(al > 0.0)) continue;
    const uint64_t N = dims[m];
    std::vector<double> cdf(N);
    double acc = 0.0;
    for (uint64_t k = 0; k < N; ++k) {
      acc += std::pow(static_cast<double>(k + 1), -al);
      cdf[k] = acc;
    }
    for (auto& c : cdf) c /= acc;
    cdf[N - 1] = 1.0;
    std::vector<uint32_t> perm(N);
    for (uint64_t k = 0; k < N; ++k) perm[k] = static_cast<uint32_t>(k);
    HostRng rng{fork64(fork64(seed, 7), m)};
    for (uint64_t k = N - 1; k > 0; --k) std::swap(perm[k], perm[rng.below(k + 1)]);
    NTCB_CUDA(cudaMalloc(&d_cdf[m], sizeof(double) * N));
    NTCB_CUDA(cudaMalloc(&d_perm[m], sizeof(uint32_t) * N));
    NTCB_CUDA(cudaMemcpy(d_cdf[m], cdf.data(), sizeof(double) * N, cudaMemcpyHostToDevice));
    NTCB_CUDA(cudaMemcpy(d_perm[m], perm.data(), sizeof(uint32_t) * N, cudaMemcpyHostToDevice));
    d.cdf[m] = d_cdf[m];
    d.perm[m] = d_perm[m];
  }

  // Candidate ids are u32 (sort payload): at most 2^32 - 2 candidates per
  // device.  Config 5 (1.7B cells of a Zipf(1.1, 1.1, 1.3) product) needs
  // ~4.05e9 of them -- the retry policy below clamps to the cap instead of
  // overshooting it, so that tensor still fits one device.
  constexpr uint64_t kMaxCand = (1ull << 32) - 2;
  uint64_t M = nnz + std::max<uint64_t>(nnz / 256, 4096);
  Buf<uint32_t> chosen(nnz);
  for (int attempt = 0;; ++attempt) {
    if (M > kMaxCand) fail(NTCB_EINVAL, "synth: too many candidates (duplicate-heavy distribution)");
    Buf<uint64_t> key(M), key2(M);
    Buf<uint32_t> jj(M), jj2(M);
    k_candidates<<<grid_of(M, sms), 256, 0, st>>>(s_mask, M, d, key.p, jj.p);
    NTCB_CUDA(cudaGetLastError());
    cub::DoubleBuffer<uint64_t> dk(key.p, key2.p);
    cub::DoubleBuffer<uint32_t> dv(jj.p, jj2.p);
    size_t tmp = 0;
    NTCB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, static_cast<int64_t>(M), 0, bits, st));
    Buf<unsigned char> t(tmp);
    NTCB_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, dk, dv, static_cast<int64_t>(M), 0, bits, st));
    Buf<unsigned long long> cnt(1);
    NTCB_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
    uint32_t* keep = dv.Current() == jj.p ? jj2.p : jj.p;
    k_first<<<grid_of(M, sms), 256, 0, st>>>(dk.Current(), dv.Current(), M, keep, cnt.p);
    NTCB_CUDA(cudaGetLastError());
    unsigned long long uniq = 0;
    NTCB_CUDA(cudaMemcpyAsync(&uniq, cnt.p, sizeof uniq, cudaMemcpyDeviceToHost, st));
    NTCB_CUDA(cudaStreamSynchronize(st));
    if (uniq < nnz) {
      const double frac = static_cast<double>(uniq) / static_cast<double>(M);
      uint64_t next = static_cast<uint64_t>(static_cast<double>(nnz) / std::max(frac, 1e-3) * 1.05) + 4096;
      next = std::max<uint64_t>(next, M + M / 4);
      // the unique fraction falls as M grows: one last try at the cap
      if (next > kMaxCand && M < kMaxCand) next = kMaxCand;
      M = next;
      continue;
    }
    // ascending j; skipped entries carry 0xffffffff and sort last
    uint32_t* other = dv.Current();
    size_t tmp2 = 0;
    NTCB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp2, keep, other, static_cast<int64_t>(M), 0, 32, st));
    Buf<unsigned char> t2(tmp2);
    NTCB_CUDA(cub::DeviceRadixSort::SortKeys(t2.p, tmp2, keep, other, static_cast<int64_t>(M), 0, 32, st));
    NTCB_CUDA(cudaMemcpyAsync(chosen.p, other, sizeof(uint32_t) * nnz, cudaMemcpyDeviceToDevice, st));
    NTCB_CUDA(cudaStreamSynchronize(st));
    break;
  }

  const int R = static_cast<int>(true_rank);
  std::vector<double*> truth(order, nullptr);
  struct TruthCleanup {
    std::vector<double*>& t;
    ~TruthCleanup() {
      for (double* p : t)
        if (p) cudaFree(p);
    }
  } truth_cleanup{truth};
  for (int m = 0; m < order; ++m) {
    NTCB_CUDA(cudaMalloc(&truth[m], sizeof(double) * dims[m] * R));
    k_truth<<<grid_of(dims[m] * R, sms), 256, 0, st>>>(fork64(fork64(seed, 4), m), dims[m] * R,
                                                       truth[m]);
    NTCB_CUDA(cudaGetLastError());
  }
  Buf<double*> dtruth(NTCB_MAX_ORDER);
  NTCB_CUDA(cudaMemcpyAsync(dtruth.p, truth.data(), sizeof(double*) * order, cudaMemcpyHostToDevice, st));
  Buf<uint32_t> idx(nnz * order);
  Buf<float> vals(nnz);
  k_emit<<<grid_of(nnz, sms), 256, 0, st>>>(chosen.p, nnz, s_mask, d, R, dtruth.p, noise_root,
                                            sigma, kind, idx.p, vals.p);
  NTCB_CUDA(cudaGetLastError());
  NTCB_CUDA(cudaStreamSynchronize(st));
  for (double*& p : truth) {
    cudaFree(p);
    p = nullptr;
  }
  chosen.release();  // the tensor build of a 1.7B-entry tensor needs the room
  load_tensor_f32(ctx, order, dims, nnz, idx.p, vals.p, true);
}

void synth_uniform(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                   uint64_t true_rank, double sigma, uint64_t seed) {
  synth_general(ctx, order, dims, nnz, true_rank, sigma, seed, nullptr, 0);
}

}  // namespace ntcb
