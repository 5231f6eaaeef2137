// Masked SSE / sum x^2 / sum ||U||^2 over Omega: the device form of
// objective() and relative_error() (metrics.cpp:8-37) with cpd_value()
// (factor_set.cpp:72-86) fused in.  The reference evaluates these serially;
// here every entry of the mode-0 view (= the canonical lexicographic order)
// is one thread, model values are formed in fp64 from the fp32 factors, and
// the per-block fp64 partials are reduced in a fixed order (deterministic).
#include <algorithm>

#include "common.cuh"

namespace ntcb {

namespace {

constexpr int kMT = 256;
constexpr int kPerThread = 8;

__device__ __forceinline__ uint64_t row_of(const uint64_t* off, uint64_t lo, uint64_t hi,
                                           uint64_t e) {
  // last row p in [lo, hi] with off[p] <= e
  while (lo < hi) {
    const uint64_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= e)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kMT) k_sse(const uint64_t* off, uint64_t rows,
                                             const uint32_t* const* oth, const float* val,
                                             uint64_t nnz, FactorArgs f, double* part) {
  __shared__ uint64_t bounds[2];
  __shared__ double red[2][kMT / 32];
  const uint64_t e0 = static_cast<uint64_t>(blockIdx.x) * kMT * kPerThread;
  const uint64_t e1 = (nnz < e0 + static_cast<uint64_t>(kMT) * kPerThread) ? nnz : e0 + static_cast<uint64_t>(kMT) * kPerThread;
  if (threadIdx.x < 2) {
    const uint64_t e = threadIdx.x == 0 ? e0 : (e1 > 0 ? e1 - 1 : 0);
    bounds[threadIdx.x] = row_of(off, 0, rows - 1, e);
  }
  __syncthreads();
  double sse = 0.0, sx = 0.0;
  const int R = f.rank, ld = f.ld;
  for (uint64_t e = e0 + threadIdx.x; e < e1; e += kMT) {
    const uint64_t p = row_of(off, bounds[0], bounds[1], e);
    const double x = static_cast<double>(val[e]);
    double model = 0.0;
    for (int r = 0; r < R; ++r) {
      double prod = static_cast<double>(f.U[0][p * ld + r]);
      for (int m = 1; m < f.order; ++m)
        prod *= static_cast<double>(f.U[m][static_cast<uint64_t>(oth[m - 1][e]) * ld + r]);
      model += prod;
    }
    const double d = x - model;
    sse += d * d;
    sx += x * x;
  }
  for (int o = 16; o; o >>= 1) {
    sse += __shfl_xor_sync(0xffffffffu, sse, o);
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = sse;
    red[1][threadIdx.x >> 5] = sx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kMT / 32; ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

__global__ void k_sumsq(const float* u, uint64_t n, double* part) {
  __shared__ double red[kMT / 32];
  double s = 0.0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(kMT) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * kMT) {
    const double v = static_cast<double>(u[i]);
    s += v * v;
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < kMT / 32; ++w) a += red[w];
    part[blockIdx.x] = a;
  }
}

// fixed-order final reduction: out[c] = sum_i part[i*stride + c]
__global__ void k_final(const double* part, uint64_t n, int stride, double* out) {
  __shared__ double red[kMT];
  for (int c = 0; c < stride; ++c) {
    double s = 0.0;
    for (uint64_t i = threadIdx.x; i < n; i += kMT) s += part[i * stride + c];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = kMT / 2; w; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[c] = red[0];
    __syncthreads();
  }
}

}  // namespace

void device_metrics(ntcb_context* ctx, double* sse, double* sumsq, double* reg) {
  cudaStream_t st = ctx->stream;
  const uint64_t nnz = ctx->nnz;
  const uint64_t blocks = (nnz + kMT * kPerThread - 1) / (kMT * kPerThread);
  const uint64_t need = 2 * std::max<uint64_t>(blocks, 1) + 64 * 16 + 8;
  if (ctx->red_n < need) {
    if (ctx->red) cudaFree(ctx->red);
    NTCB_CUDA(cudaMalloc(&ctx->red, sizeof(double) * need));
    ctx->red_n = need;
  }
  double* part = ctx->red;
  double* outs = ctx->red + ctx->red_n - 8;
  double h[3] = {0, 0, 0};
  if (nnz) {
    FactorArgs f{};
    for (int m = 0; m < ctx->order; ++m) f.U[m] = ctx->A[m];
    f.order = ctx->order;
    f.mode = 0;
    f.rank = static_cast<int>(ctx->rank);
    f.ld = static_cast<int>(ctx->ld);
    // stage the SoA pointer table in device memory (8 doubles after the partials)
    static_assert(sizeof(uint32_t*) == 8, "64-bit");
    uint32_t* tbl[NTCB_MAX_ORDER] = {};
    for (int k = 0; k < ctx->order - 1; ++k) tbl[k] = ctx->views[0].oth[k];
    uint32_t** dt = reinterpret_cast<uint32_t**>(part + 2 * blocks);
    NTCB_CUDA(cudaMemcpyAsync(dt, tbl, sizeof tbl, cudaMemcpyHostToDevice, st));
    const uint32_t* const* oth = dt;
    k_sse<<<static_cast<unsigned>(blocks), kMT, 0, st>>>(ctx->views[0].off, ctx->views[0].rows,
                                                         oth, ctx->views[0].val, nnz, f, part);
    NTCB_CUDA(cudaGetLastError());
    k_final<<<1, kMT, 0, st>>>(part, blocks, 2, outs);
    NTCB_CUDA(cudaGetLastError());
    NTCB_CUDA(cudaMemcpyAsync(h, outs, sizeof(double) * 2, cudaMemcpyDeviceToHost, st));
    NTCB_CUDA(cudaStreamSynchronize(st));
  }
  double rg = 0.0;
  for (int m = 0; m < ctx->order; ++m) {
    const uint64_t n = ctx->dims[m] * ctx->ld;
    const unsigned g = static_cast<unsigned>(std::min<uint64_t>((n + kMT - 1) / kMT, 64));
    k_sumsq<<<g, kMT, 0, st>>>(ctx->A[m], n, part + 2 * blocks + 16);
    NTCB_CUDA(cudaGetLastError());
    k_final<<<1, kMT, 0, st>>>(part + 2 * blocks + 16, g, 1, outs + 2);
    NTCB_CUDA(cudaGetLastError());
    double v = 0.0;
    NTCB_CUDA(cudaMemcpyAsync(&v, outs + 2, sizeof(double), cudaMemcpyDeviceToHost, st));
    NTCB_CUDA(cudaStreamSynchronize(st));
    rg += v;
  }
  *sse = h[0];
  *sumsq = h[1];
  *reg = rg;
}

}  // namespace ntcb
