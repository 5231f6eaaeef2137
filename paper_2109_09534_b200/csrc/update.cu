// Row update of S_NMC (nmc.cpp:199-272 minus sampling): for every processed
// row p of view `mode`, one CTA
//   1. streams the slice's entries (coalesced SoA loads) and keeps the ones
//      whose bit is set in the sampled-set mask (all of them at c >= 1);
//   2. for each kept entry builds the augmented Khatri-Rao row
//      k~ = [k_1..k_R, s], k = Hadamard product of the other factors' rows
//      (kr_row, factor_set.cpp:42-64), s = y.k - x (residual at Y);
//   3. accumulates the Gram matrix  sum k~ k~^T  with a register-tiled 4x4
//      outer-product scheme: its R x R block is the sampled Hessian minus
//      lambda I and its last column is w + z (nmc.cpp:68-106);
//   4. finalises on warp 0 in fp64: H = lambda I + sum k k^T, grad =
//      sum s k + lambda y, finiteness checks, power method from the
//      normalised all-ones vector (nmc.cpp:140-172), L = 1.01 * rq
//      (nmc.cpp:253-254), projected step + Nesterov momentum (nmc.cpp:174-197).
// fp32 accumulation, fp64 finalisation.  Summation is in slice order rather
// than draw order (same sampled set, bit-exact; sums agree to fp32 rounding).
#include "common.cuh"

namespace ntcb {

struct UpdateArgs {
  const uint64_t* off;
  const uint32_t* oth[NTCB_MAX_ORDER - 1];
  const float* val;
  const uint32_t* mask;
  FactorArgs f;
  float* A;  // factors[mode]
  float* Y;  // momentum[mode]
  uint64_t row_begin, row_end;
  double c;
  double lambda;
  double power_tol;
  int power_iters;
  unsigned long long* counters;
};

constexpr int kThreads = 256;
constexpr int kTile = 512;  // entries examined per tile (2 per thread)

__device__ __forceinline__ void report(unsigned long long* counters, int mode, uint64_t row,
                                       int kind) {
  const unsigned long long key =
      (static_cast<unsigned long long>(mode) << 58) | (static_cast<unsigned long long>(row) << 2) |
      static_cast<unsigned long long>(kind);
  atomicMin(&counters[1], key);
}

template <int RP>
__global__ void __launch_bounds__(kThreads, 2) k_update(UpdateArgs a) {
  constexpr int NB4 = RP / 4;
  constexpr int NBLK = NB4 * (NB4 + 1) / 2;
  constexpr int G = (kThreads / NBLK) >= 1 ? (kThreads / NBLK) : 1;
  extern __shared__ __align__(16) unsigned char smem[];
  float* K = reinterpret_cast<float*>(smem);                // kTile x RP
  float* red = K + kTile * RP;                              // G x NBLK x 16 (<= 4096 floats)
  double* Hd = reinterpret_cast<double*>(red + kThreads * 16);  // R x HS (HS odd stride)
  const int R = a.f.rank;
  const int HS = R | 1;
  double* gd = Hd + R * HS;        // gradient (R)
  double* vv = gd + 64;            // power-method iterate (R)
  float* ys = reinterpret_cast<float*>(vv + 64);  // y row, padded to RP
  int* sidx = reinterpret_cast<int*>(ys + RP);    // kTile selected local indices
  int* wtot = sidx + kTile;                       // per-warp counts (8) + scratch

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int wid = tid >> 5;
  const int ld = a.f.ld;
  const bool full = a.c >= 1.0;

  // this thread's 4x4 block of the (RP x RP) upper triangle, and its pick group
  const int grp = tid / NBLK;
  const int blk = tid - grp * NBLK;
  const bool acc_on = grp < G;
  int bi = 0, bj = 0;
  {
    int rem = blk;
    for (int i = 0; i < NB4; ++i) {
      const int cnt = NB4 - i;
      if (rem < cnt) {
        bi = i;
        bj = i + rem;
        break;
      }
      rem -= cnt;
    }
  }

  // other modes' factor pointers in ascending mode order (kr_row order)
  const float* U[NTCB_MAX_ORDER - 1];
  int no = 0;
  for (int m = 0; m < a.f.order; ++m)
    if (m != a.f.mode) U[no++] = a.f.U[m];
  const int ld4 = ld / 4;

  for (uint64_t p = a.row_begin + blockIdx.x; p < a.row_end; p += gridDim.x) {
    if (*reinterpret_cast<volatile unsigned long long*>(&a.counters[1]) != ~0ull) return;
    const uint64_t beg = a.off[p];
    const uint64_t n = a.off[p + 1] - beg;
    const uint64_t b = blocksize_for(a.c, n);
    if (b == 0) continue;  // skipped row: A and Y untouched (nmc.cpp:237)

    if (tid < RP) ys[tid] = tid < R ? a.Y[p * ld + tid] : 0.f;
    float acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = 0.f;
    __syncthreads();

    for (uint64_t t0 = 0; t0 < n; t0 += kTile) {
      // ---- 1. selection + block compaction ------------------------------
      bool sel[2];
      int cnt = 0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint64_t t = t0 + 2 * tid + e;
        bool s = t < n;
        if (s && !full) {
          const uint64_t gb = beg + t;
          s = (__ldg(&a.mask[gb >> 5]) >> (gb & 31u)) & 1u;
        }
        sel[e] = s;
        cnt += s;
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) wtot[wid] = incl;
      __syncthreads();
      int wbase = 0, nsel = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) {
        const int v = wtot[w];
        wbase += (w < wid) ? v : 0;
        nsel += v;
      }
      int slot = wbase + incl - cnt;
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (sel[e]) sidx[slot++] = 2 * tid + e;
      __syncthreads();

      // ---- 2. gather + augmented Khatri-Rao rows --------------------------
      for (int s = tid; s < nsel; s += kThreads) {
        const uint64_t t = beg + t0 + sidx[s];
        float k[RP];
        {
          const float4* r0 = reinterpret_cast<const float4*>(U[0] + static_cast<uint64_t>(__ldg(&a.oth[0][t])) * ld);
#pragma unroll
          for (int q = 0; q < RP / 4; ++q) {
            float4 v = (q < ld4) ? __ldg(r0 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            k[4 * q] = v.x;
            k[4 * q + 1] = v.y;
            k[4 * q + 2] = v.z;
            k[4 * q + 3] = v.w;
          }
        }
        for (int m = 1; m < no; ++m) {
          const float4* rm = reinterpret_cast<const float4*>(U[m] + static_cast<uint64_t>(__ldg(&a.oth[m][t])) * ld);
#pragma unroll
          for (int q = 0; q < RP / 4; ++q) {
            if (q < ld4) {
              const float4 v = __ldg(rm + q);
              k[4 * q] *= v.x;
              k[4 * q + 1] *= v.y;
              k[4 * q + 2] *= v.z;
              k[4 * q + 3] *= v.w;
            }
          }
        }
        float dot = 0.f;
#pragma unroll
        for (int r = 0; r < RP; ++r) dot = fmaf(ys[r], k[r], dot);
        const float x = __ldg(&a.val[t]);
#pragma unroll
        for (int r = 0; r < RP; ++r)
          if (r >= R) k[r] = (r == R) ? (dot - x) : 0.f;
        float4* dst = reinterpret_cast<float4*>(K + s * RP);
#pragma unroll
        for (int q = 0; q < RP / 4; ++q)
          dst[q] = make_float4(k[4 * q], k[4 * q + 1], k[4 * q + 2], k[4 * q + 3]);
      }
      __syncthreads();

      // ---- 3. register-tiled Gram accumulation ---------------------------
      if (acc_on) {
        const float4* K4 = reinterpret_cast<const float4*>(K);
        for (int s = grp; s < nsel; s += G) {
          const float4 u = K4[s * NB4 + bi];
          const float4 w = K4[s * NB4 + bj];
          const float ua[4] = {u.x, u.y, u.z, u.w};
          const float wa[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[4 * i + j] = fmaf(ua[i], wa[j], acc[4 * i + j]);
        }
      }
      __syncthreads();
    }

    // ---- 4. reduce the pick groups, assemble H (fp64) and grad --------------
    if (acc_on) {
#pragma unroll
      for (int q = 0; q < 16; ++q) red[(grp * NBLK + blk) * 16 + q] = acc[q];
    }
    __syncthreads();
    const double lam = a.lambda;
    for (int idx = tid; idx < NBLK * 16; idx += kThreads) {
      const int bk = idx >> 4, q = idx & 15;
      float s = 0.f;
      for (int g = 0; g < G; ++g) s += red[(g * NBLK + bk) * 16 + q];
      int rem = bk, ci = 0, cj = 0;
      for (int i = 0; i < NB4; ++i) {
        const int cn = NB4 - i;
        if (rem < cn) {
          ci = i;
          cj = i + rem;
          break;
        }
        rem -= cn;
      }
      const int row = 4 * ci + (q >> 2), col = 4 * cj + (q & 3);
      if (row < R && col < R) {
        if (row <= col) {
          const double hv = static_cast<double>(s) + (row == col ? lam : 0.0);
          Hd[row * HS + col] = hv;
          Hd[col * HS + row] = hv;
        }
      } else if (row < R && col == R) {
        gd[row] = static_cast<double>(s) + lam * static_cast<double>(ys[row]);
      }
    }
    __syncthreads();

    // ---- 5. warp 0: checks, power method, projected Nesterov step ---------
    if (wid == 0) {
      bool bad = false;
      for (int r = lane; r < R; r += 32) bad |= !isfinite(gd[r]);
      if (__any_sync(0xffffffffu, bad)) {
        if (lane == 0) report(a.counters, a.f.mode, p, 0);  // non-finite gradient
      } else {
        bool hbad = false;
        for (int i = lane; i < R * R; i += 32) hbad |= !isfinite(Hd[(i / R) * HS + (i % R)]);
        if (__any_sync(0xffffffffu, hbad)) {
          if (lane == 0) report(a.counters, a.f.mode, p, 1);  // power_method rejects H
        } else {
          const double v0 = 1.0 / sqrt(static_cast<double>(R));
          for (int r = lane; r < R; r += 32) vv[r] = v0;
          __syncwarp();
          double rq = 0.0, rq_prev = 0.0;
          for (int it = 0; it < a.power_iters; ++it) {
            double u0 = 0.0, u1 = 0.0;
            if (lane < R) {
              const double* hr = Hd + lane * HS;
              for (int j = 0; j < R; ++j) u0 += hr[j] * vv[j];
            }
            if (lane + 32 < R) {
              const double* hr = Hd + (lane + 32) * HS;
              for (int j = 0; j < R; ++j) u1 += hr[j] * vv[j];
            }
            double num = 0.0, un2 = u0 * u0 + u1 * u1;
            if (lane < R) num += vv[lane] * u0;
            if (lane + 32 < R) num += vv[lane + 32] * u1;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
              num += __shfl_xor_sync(0xffffffffu, num, o);
              un2 += __shfl_xor_sync(0xffffffffu, un2, o);
            }
            rq = num;
            if (un2 == 0.0) {
              rq = 0.0;
              break;
            }
            if (it > 0 && fabs(rq - rq_prev) <= a.power_tol * fabs(rq)) break;
            rq_prev = rq;
            const double inv = 1.0 / sqrt(un2);
            __syncwarp();
            if (lane < R) vv[lane] = u0 * inv;
            if (lane + 32 < R) vv[lane + 32] = u1 * inv;
            __syncwarp();
          }
          const double L = rq * 1.01;  // nmc.cpp:253-254
          if (!(L >= lam)) {
            if (lane == 0) report(a.counters, a.f.mode, p, 2);  // row_step rejects L
          } else {
            const double inv_l = 1.0 / L;
            const double sl = sqrt(L), sm = sqrt(lam);
            const double beta = (sl - sm) / (sl + sm);
            for (int r = lane; r < R; r += 32) {
              const double y = static_cast<double>(ys[r]);
              const double ap = static_cast<double>(a.A[p * ld + r]);
              const double av = y - inv_l * gd[r];
              const double an = av > 0.0 ? av : 0.0;
              a.A[p * ld + r] = static_cast<float>(an);
              a.Y[p * ld + r] = static_cast<float>(an + beta * (an - ap));
            }
          }
        }
      }
    }
    __syncthreads();
  }
}

template <int RP>
static size_t update_smem(int R) {
  const int HS = R | 1;
  return static_cast<size_t>(kTile) * RP * 4 + kThreads * 16 * 4 +
         static_cast<size_t>(R) * HS * 8 + 64 * 8 * 2 + RP * 4 + kTile * 4 + 64 * 4;
}

template <int RP>
static void launch_rp(ntcb_context* ctx, const UpdateArgs& a, uint64_t rows) {
  const size_t smem = update_smem<RP>(a.f.rank);
  NTCB_CUDA(cudaFuncSetAttribute(k_update<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  int per_sm = 0;
  NTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_update<RP>, kThreads, smem));
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = rows;
  const uint64_t cap = static_cast<uint64_t>(per_sm) * ctx->sm_count;
  if (grid > cap) grid = cap;
  k_update<RP><<<static_cast<unsigned>(grid), kThreads, smem, ctx->stream>>>(a);
  NTCB_CUDA(cudaGetLastError());
}

int launch_update(ntcb_context* ctx, int mode, uint64_t row_begin, uint64_t row_end,
                  const ntcb_nmc_config& cfg) {
  if (row_end <= row_begin) return 0;
  const DeviceView& v = ctx->views[mode];
  UpdateArgs a{};
  a.off = v.off;
  for (int k = 0; k < ctx->order - 1; ++k) a.oth[k] = v.oth[k];
  a.val = v.val;
  a.mask = ctx->mask;
  for (int m = 0; m < ctx->order; ++m) a.f.U[m] = ctx->A[m];
  a.f.order = ctx->order;
  a.f.mode = mode;
  a.f.rank = static_cast<int>(ctx->rank);
  a.f.ld = static_cast<int>(ctx->ld);
  a.A = ctx->A[mode];
  a.Y = ctx->Y[mode];
  a.row_begin = row_begin;
  a.row_end = row_end;
  a.c = cfg.c;
  a.lambda = cfg.lambda;
  a.power_tol = cfg.power_tol;
  a.power_iters = cfg.power_iters;
  a.counters = ctx->counters;
  const int RP = static_cast<int>((ctx->rank + 1 + 3) / 4 * 4);
  const uint64_t rows = row_end - row_begin;
  switch (RP) {
#define NTCB_RP(x) \
  case x:          \
    launch_rp<x>(ctx, a, rows); \
    break;
    NTCB_RP(4) NTCB_RP(8) NTCB_RP(12) NTCB_RP(16) NTCB_RP(20) NTCB_RP(24) NTCB_RP(28)
    NTCB_RP(32) NTCB_RP(36) NTCB_RP(40) NTCB_RP(44) NTCB_RP(48) NTCB_RP(52) NTCB_RP(56)
    NTCB_RP(60) NTCB_RP(64) NTCB_RP(68)
#undef NTCB_RP
    default:
      fail(NTCB_EINVAL, "s_nmc: rank exceeds the supported maximum (64)");
  }
  return 1;
}

}  // namespace ntcb
