// Masked SSE / sum x^2 / sum ||U||^2 over Omega: the device form of
// objective() and relative_error() (metrics.cpp:8-37) with cpd_value()
// (factor_set.cpp:72-86) fused in.
//
// The mode-0 view (= the canonical lexicographic order) is cut into items of
// <= kItem entries of one row; a warp takes an item: the row's own factor
// row is loaded once, then 4 entries per step, 8 lanes per entry, a lane
// holding 4 features (16-byte loads of each other factor's row: one 128-byte
// line per entry and factor for ranks <= 32).  Model values and the squares
// are fp64 (products of the fp32 factors are exact in fp64 up to 3 factors).
// Per-item partials are reduced in item order by one CTA (deterministic).
#include <algorithm>
#include <map>
#include <vector>

#include "common.cuh"

namespace ntcb {

namespace {

constexpr int kMT = 256;
constexpr uint32_t kItem = 4096;  // entries per item

struct MItem {
  uint64_t row, e0, e1;
};

struct MArgs {
  const MItem* items;
  uint64_t n_items;
  const uint32_t* oth[NTCB_MAX_ORDER - 1];
  const float* val;
  const float* U[NTCB_MAX_ORDER];  // U[0] = the mode-0 factor, then the others in mode order
  int no;
  int rank;
  int ld;
  double* part;  // [item][2]: sse, sum x^2
};

constexpr int kSteps = 4;  // steps of 4 entries with their gathers in flight together

__device__ __forceinline__ const float4* row4(const float* base, uint32_t row, uint32_t ld4) {
  uint64_t p;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(row), "r"(ld4), "l"(reinterpret_cast<uint64_t>(base)));
  return reinterpret_cast<const float4*>(p);
}

template <int NC, int NO>  // feature chunks of 32 (rank <= 32 * NC); other modes (NO < max: exact)
__global__ void __launch_bounds__(kMT, 2) k_sse(MArgs a) {
  const int lane = threadIdx.x & 31;
  const int grp = lane >> 3, sub = lane & 7;  // entry slot, feature quad
  const int no = NO < NTCB_MAX_ORDER - 1 ? NO : a.no;
  const uint32_t ld4 = static_cast<uint32_t>(a.ld) * 4u;
  // lane base of every other factor: feature 4*sub (+32 per chunk); reads past
  // the row (rank < 32) hit the next row or the 32-float slack and meet a
  // zero in the mode-0 row
  const float* ub[NO > 0 ? NO : 1];
#pragma unroll
  for (int m = 0; m < NO; ++m) ub[m] = a.U[(m < no ? m : 0) + 1] + 4 * sub;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (kMT / 32);
  for (uint64_t it = blockIdx.x * static_cast<uint64_t>(kMT / 32) + (threadIdx.x >> 5); it < a.n_items; it += nw) {
    const MItem w = a.items[it];
    double ad[NC][4];  // this row's mode-0 factor features, fp64; 0 beyond R
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int f = 32 * c + 4 * sub;
      const float4 v = __ldg(reinterpret_cast<const float4*>(a.U[0] + w.row * a.ld + f));
      ad[c][0] = f + 0 < a.rank ? static_cast<double>(v.x) : 0.0;
      ad[c][1] = f + 1 < a.rank ? static_cast<double>(v.y) : 0.0;
      ad[c][2] = f + 2 < a.rank ? static_cast<double>(v.z) : 0.0;
      ad[c][3] = f + 3 < a.rank ? static_cast<double>(v.w) : 0.0;
    }
    double sse = 0.0, sx = 0.0;
    // 32 entries per round: one coalesced load of their coordinates and
    // values (the next round's issued before this round's gathers), then
    // steps of 4 entries whose factor-row gathers are in flight together
    // (coordinates move to the lanes by shuffles)
    uint32_t idx[NO > 0 ? NO : 1], nidx[NO > 0 ? NO : 1];
    float xv, nxv = 0.f;
    auto load_round = [&](uint64_t b0, uint32_t* ix, float& x) {
      const uint64_t eb = b0 + lane;
      const bool inb = eb < w.e1;
#pragma unroll
      for (int m = 0; m < NO; ++m)
        if (m < no) ix[m] = inb ? __ldg(a.oth[m] + eb) : 0u;
      x = inb ? __ldg(a.val + eb) : 0.f;
    };
    load_round(w.e0, idx, xv);
    for (uint64_t b0 = w.e0; b0 < w.e1; b0 += 32) {
      if (b0 + 32 < w.e1) load_round(b0 + 32, nidx, nxv);
#pragma unroll 1
      for (int u0 = 0; u0 < 8; u0 += kSteps) {
        float4 v[kSteps][NC][NO > 0 ? NO : 1];
#pragma unroll
        for (int uu = 0; uu < kSteps; ++uu) {
#pragma unroll
          for (int m = 0; m < NO; ++m)
            if (m < no) {
              const uint32_t row = __shfl_sync(0xffffffffu, idx[m], 4 * (u0 + uu) + grp);
              const float4* rp = row4(ub[m], row, ld4);
#pragma unroll
              for (int c = 0; c < NC; ++c) v[uu][c][m] = __ldg(rp + 8 * c);
            }
        }
#pragma unroll
        for (int uu = 0; uu < kSteps; ++uu) {
          const int u = u0 + uu;
          double part = 0.0;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            double p0 = ad[c][0], p1 = ad[c][1], p2 = ad[c][2], p3 = ad[c][3];
#pragma unroll
            for (int m = 0; m < NO; ++m)
              if (m < no) {
                p0 *= v[uu][c][m].x;
                p1 *= v[uu][c][m].y;
                p2 *= v[uu][c][m].z;
                p3 *= v[uu][c][m].w;
              }
            part += (p0 + p1) + (p2 + p3);
          }
#pragma unroll
          for (int o = 4; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
          const double x = static_cast<double>(__shfl_sync(0xffffffffu, xv, 4 * u + grp));
          if (sub == 0 && b0 + 4 * u + grp < w.e1) {
            const double d = x - part;
            sse += d * d;
            sx += x * x;
          }
        }
      }
#pragma unroll
      for (int m = 0; m < NO; ++m) idx[m] = nidx[m];
      xv = nxv;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      sse += __shfl_xor_sync(0xffffffffu, sse, o);
      sx += __shfl_xor_sync(0xffffffffu, sx, o);
    }
    if (lane == 0) {
      a.part[2 * it] = sse;
      a.part[2 * it + 1] = sx;
    }
  }
}

// sum of squares of every factor (padding is zero), one partial per block
__global__ void k_sumsq(const float* const* U, const uint64_t* n, int order, double* part) {
  __shared__ double red[kMT / 32];
  double s = 0.0;
  for (int m = 0; m < order; ++m)
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(kMT) + threadIdx.x; i < n[m];
         i += static_cast<uint64_t>(gridDim.x) * kMT) {
      const double v = static_cast<double>(U[m][i]);
      s += v * v;
    }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kMT / 32; ++w) t += red[w];
    part[blockIdx.x] = t;
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

struct MPlan {
  MItem* items = nullptr;
  uint64_t n = 0;
};
using MPlans = std::map<const void*, MPlan>;

const MPlan& mplan(ntcb_context* ctx) {
  auto& g_mplans = ctx_cache<MPlans>(ctx, kCacheMetrics);
  const DeviceView& v = ctx->views[0];
  auto it = g_mplans.find(v.off);
  if (it != g_mplans.end()) return it->second;
  // items of <= kItem entries, shorter when the tensor is small (~2 per warp slot)
  const uint64_t nnz = v.h_off[v.rows];
  const uint64_t slots = static_cast<uint64_t>(ctx->sm_count) * 32;
  const uint64_t len = std::min<uint64_t>(kItem, std::max<uint64_t>(256, (nnz / (2 * slots) + 31) / 32 * 32));
  std::vector<MItem> items;
  for (uint64_t p = v.row_lo; p < v.row_hi; ++p)  // resident rows (a slab on a multi-GPU shard)
    for (uint64_t e = v.h_off[p]; e < v.h_off[p + 1]; e += len)
      items.push_back({p, e, std::min<uint64_t>(v.h_off[p + 1], e + len)});
  MPlan pl;
  pl.n = items.size();
  if (pl.n) {
    NTCB_CUDA(cudaMalloc(&pl.items, sizeof(MItem) * pl.n));
    NTCB_CUDA(cudaMemcpy(pl.items, items.data(), sizeof(MItem) * pl.n, cudaMemcpyHostToDevice));
  }
  return g_mplans.emplace(v.off, pl).first->second;
}

}  // namespace

void drop_metric_plans(ntcb_context* ctx) {
  if (!ctx->cache[kCacheMetrics]) return;
  for (auto& kv : ctx_cache<MPlans>(ctx, kCacheMetrics))
    if (kv.second.items) cudaFree(kv.second.items);
  ctx_cache_free<MPlans>(ctx, kCacheMetrics);
}

void device_metrics(ntcb_context* ctx, double* sse, double* sumsq, double* reg) {
  cudaStream_t st = ctx->stream;
  const MPlan& pl = mplan(ctx);
  const unsigned sq_blocks = 64;
  // partials: [items][2] | sumsq [64] | table of factor pointers and sizes | outputs [3]
  const uint64_t need = 2 * std::max<uint64_t>(pl.n, 1) + sq_blocks + 4 * NTCB_MAX_ORDER + 8;
  if (ctx->red_n < need) {
    if (ctx->red) cudaFree(ctx->red);
    NTCB_CUDA(cudaMalloc(&ctx->red, sizeof(double) * need));
    ctx->red_n = need;
  }
  double* part = ctx->red;
  double* sq = part + 2 * std::max<uint64_t>(pl.n, 1);
  double* tblmem = sq + sq_blocks;
  double* outs = ctx->red + ctx->red_n - 8;
  // factor pointer / size tables for k_sumsq (staged in device memory)
  struct {
    const float* U[NTCB_MAX_ORDER];
    uint64_t n[NTCB_MAX_ORDER];
  } tbl{};
  for (int m = 0; m < ctx->order; ++m) {
    tbl.U[m] = ctx->A[m];
    tbl.n[m] = ctx->dims[m] * ctx->ld;
  }
  static_assert(sizeof(tbl) <= sizeof(double) * 4 * NTCB_MAX_ORDER, "table fits");
  NTCB_CUDA(cudaMemcpyAsync(tblmem, &tbl, sizeof tbl, cudaMemcpyHostToDevice, st));
  if (pl.n) {
    MArgs a{};
    a.items = pl.items;
    a.n_items = pl.n;
    for (int k = 0; k < ctx->order - 1; ++k) a.oth[k] = ctx->views[0].oth[k];
    a.val = ctx->views[0].val;
    for (int m = 0; m < ctx->order; ++m) a.U[m] = ctx->A[m];
    a.no = ctx->order - 1;
    a.rank = static_cast<int>(ctx->rank);
    a.ld = static_cast<int>(ctx->ld);
    a.part = part;
    const uint64_t warps = std::min<uint64_t>(pl.n, static_cast<uint64_t>(ctx->sm_count) * 32);
    const unsigned grid = static_cast<unsigned>((warps + kMT / 32 - 1) / (kMT / 32));
    const bool wide = ctx->ld > 32;
    switch (a.no) {
#define NTCB_SSE(NO_)                                              \
  case NO_:                                                        \
    if (wide)                                                      \
      k_sse<2, NO_><<<grid, kMT, 0, st>>>(a);                      \
    else                                                           \
      k_sse<1, NO_><<<grid, kMT, 0, st>>>(a);                      \
    break;
      NTCB_SSE(1) NTCB_SSE(2) NTCB_SSE(3)
#undef NTCB_SSE
      default:
        if (wide)
          k_sse<2, NTCB_MAX_ORDER - 1><<<grid, kMT, 0, st>>>(a);
        else
          k_sse<1, NTCB_MAX_ORDER - 1><<<grid, kMT, 0, st>>>(a);
    }
    NTCB_CUDA(cudaGetLastError());
    k_final<<<1, kMT, 0, st>>>(part, pl.n, 2, outs);
    NTCB_CUDA(cudaGetLastError());
  } else {
    NTCB_CUDA(cudaMemsetAsync(outs, 0, sizeof(double) * 2, st));
  }
  const auto* t = reinterpret_cast<const decltype(tbl)*>(tblmem);
  k_sumsq<<<sq_blocks, kMT, 0, st>>>(t->U, t->n, ctx->order, sq);
  NTCB_CUDA(cudaGetLastError());
  k_final<<<1, kMT, 0, st>>>(sq, sq_blocks, 1, outs + 2);
  NTCB_CUDA(cudaGetLastError());
  double h[3] = {0, 0, 0};
  NTCB_CUDA(cudaMemcpyAsync(h, outs, sizeof h, cudaMemcpyDeviceToHost, st));
  NTCB_CUDA(cudaStreamSynchronize(st));
  *sse = h[0];
  *sumsq = h[1];
  *reg = h[2];
}

}  // namespace ntcb
