// tcgen05 Gram microbenchmark: natural-layout factor-row
// gathers (8 consecutive lanes read a pick's 128-byte row as float4) ->
// Khatri-Rao product in registers -> bf16 hi/lo split -> 128-byte-swizzled
// MN-major operand tile in shared memory -> tcgen05.mma (M 64, N 32, K 16,
// D = [hi; lo] hi^T in tensor memory), one accumulator per warp, read back
// and summed by the warpgroup at the end of an "item".
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o .mb/umma_gram tools/microbench/umma_gram.cu
//
// Part 1 checks the descriptor / swizzle / tensor-memory layout assumptions
// against a host computation (and measures the accumulation bias of long
// in-TMEM sums); part 2 measures G picks/s against the LDG pair-layout
// gather of tools/microbench/hybrid.cu (56 G picks/s) and the product kernel
// (37 G picks/s at config 2).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "umma.cuh"

using namespace ntcb::umma;

struct Pick {
  uint32_t j, k;
  float x;
  uint32_t pad;
};

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr int NT = 2;       // operand tiles per warp
constexpr int RING = 128;   // pick ring slots per warp (four blocks of 32)

template <int NO>
struct TileRegs {
  float4 a[4], b[4], c[NO == 3 ? 4 : 1];
  float x[4];
};

// ILV: accumulators of warps 2, 3 at tensor-memory lane offset 16 (64 columns
// per CTA); otherwise four column blocks (128 columns)
template <bool ILV, bool DUMP, int STAGES, int NO = 2>
__global__ void __launch_bounds__(128) k_gram(const float* __restrict__ U1, const float* __restrict__ U2,
                                              const Pick* __restrict__ picks, int ppw, int item_picks, int R,
                                              float* __restrict__ out, float* __restrict__ raw, int pad_smem) {
  extern __shared__ __align__(1024) unsigned char sm[];
  constexpr int COLS = ILV ? 64 : 128;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int oct = lane >> 3, q = lane & 7;
  unsigned char* tiles = sm + wid * NT * kTileBytes;
  uint4* ring = reinterpret_cast<uint4*>(sm + 4 * NT * kTileBytes) + wid * RING;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 4 * NT * kTileBytes + 4 * RING * 16) + wid * (NT + 1);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + 4 * NT * kTileBytes + 4 * RING * 16 + 4 * (NT + 1) * 8);
  if (pad_smem < 0) sm[threadIdx.x] = 0;
  if (lane == 0) {
    for (int b = 0; b <= NT; ++b) mbar_init(&bars[b], 1);
  }
  if (wid == 0) tmem_alloc<COLS>(tslot);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = *tslot;
  const uint32_t dacc = ILV ? tbase + (static_cast<uint32_t>(16 * (wid >> 1)) << 16) + 32u * (wid & 1) : tbase + 32u * wid;
  const uint32_t idesc = idesc_bf16(64, 32);
  const int QN = (R + 1 + 3) / 4;  // float4 chunks that hold features 0..R
  const int XQ = R >> 2, XC = R & 3;

  const int gwarp = blockIdx.x * 4 + wid;
  const Pick* mine = picks + static_cast<size_t>(gwarp) * ppw;
  const int n_items = ppw / item_picks;
  uint32_t gtile = 0;       // tiles issued by this warp so far
  uint32_t done_phase = 0;

  auto load_tile = [&](TileRegs<NO>& t, int rbase, int np) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int n = 4 * s + oct;
      const uint4 e = ring[(rbase + n) & (RING - 1)];
      const bool on = n < np && q < QN;
      t.a[s] = on ? __ldg(reinterpret_cast<const float4*>(U1 + static_cast<size_t>(e.x) * 32) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      t.b[s] = on ? __ldg(reinterpret_cast<const float4*>(U2 + static_cast<size_t>(e.y) * 32) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (NO == 3)
        t.c[s] = on ? __ldg(reinterpret_cast<const float4*>(U1 + static_cast<size_t>(e.w) * 32) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      t.x[s] = n < np ? __uint_as_float(e.z) : 0.f;
    }
  };
  auto store_tile = [&](const TileRegs<NO>& t, unsigned char* tile) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      float4 k = make_float4(t.a[s].x * t.b[s].x, t.a[s].y * t.b[s].y, t.a[s].z * t.b[s].z, t.a[s].w * t.b[s].w);
      if constexpr (NO == 3) k = make_float4(k.x * t.c[s].x, k.y * t.c[s].y, k.z * t.c[s].z, k.w * t.c[s].w);
      if (q == XQ) {  // the x column of k' = (k, x, 0...)
        if (XC == 0) k = make_float4(t.x[s], 0.f, 0.f, 0.f);
        else if (XC == 1) k = make_float4(k.x, t.x[s], 0.f, 0.f);
        else if (XC == 2) k = make_float4(k.x, k.y, t.x[s], 0.f);
        else k.w = t.x[s];
      }
      uint2 hi, lo;
      split_bf16(k, hi, lo);
      tile_store(tile, tile_row_of(s, oct), q, hi, lo);
    }
  };

  for (int it = 0; it < n_items; ++it) {
    const Pick* ip = mine + static_cast<size_t>(it) * item_picks;
    const int ntile = (item_picks + 15) / 16;
    // pick ring: blocks of 32 picks (two tiles), block b at ring[(b & 3) * 32]
    uint4 nxt = lane < item_picks ? *reinterpret_cast<const uint4*>(ip + lane) : make_uint4(0, 0, 0, 0);
    int tl = 0;  // next tile to gather
    auto load_next = [&](TileRegs<NO>& r) {
      if ((tl & 1) == 0) {
        const int blk = tl >> 1;
        ring[((blk & 3) << 5) + lane] = nxt;
        if ((blk + 1) * 32 + lane < item_picks) nxt = *reinterpret_cast<const uint4*>(ip + (blk + 1) * 32 + lane);
        __syncwarp();
      }
      load_tile(r, tl * 16, min(16, item_picks - tl * 16));
      ++tl;
    };
    bool first = true;
    auto emit = [&](const TileRegs<NO>& r) {
      const uint32_t b = gtile % NT, n = gtile / NT;
      if (n >= 1) mbar_wait(&bars[b], (n - 1) & 1);  // the MMA that read this buffer is done
      unsigned char* tile = tiles + b * kTileBytes;
      store_tile(r, tile);
      fence_smem_to_async();
      __syncwarp();
      if (lane == 0) {
        fence_after_sync();
        const uint64_t d = smem_desc_mn_sw128(smem_u32(tile));
        mma_bf16_ss(dacc, d, d, idesc, first ? 0u : 1u);
        commit(&bars[b]);
      }
      first = false;
      ++gtile;
    };
    TileRegs<NO> r0, r1, r2;
    if constexpr (STAGES == 3) {
      load_next(r0);
      if (1 < ntile) load_next(r1);
      for (int t = 0; t < ntile; t += 3) {
        if (t + 2 < ntile) load_next(r2);
        emit(r0);
        if (t + 1 < ntile) {
          if (t + 3 < ntile) load_next(r0);
          emit(r1);
          if (t + 2 < ntile) {
            if (t + 4 < ntile) load_next(r1);
            emit(r2);
          }
        }
      }
    } else {
      load_next(r0);
      for (int t = 0; t < ntile; t += 2) {
        if (t + 1 < ntile) load_next(r1);
        emit(r0);
        if (t + 1 < ntile) {
          if (t + 2 < ntile) load_next(r0);
          emit(r1);
        }
      }
    }
    // item end: all of this warp's MMAs done, then the warpgroup reads back
    if (lane == 0) commit(&bars[NT]);
    mbar_wait(&bars[NT], done_phase);
    done_phase ^= 1;
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    float v[32], u[32];
    const uint32_t lane_base = tbase + (static_cast<uint32_t>(32 * wid) << 16);
    if constexpr (ILV) {
      tmem_ld32(lane_base, v);       // lanes < 16: warp-0 accumulator; >= 16: warp 2's
      tmem_ld32(lane_base + 32, u);  // warp 1 / warp 3
      if constexpr (DUMP) {
        float* rr = raw + (static_cast<size_t>(blockIdx.x) * n_items + it) * 128 * 128 + (32 * wid + lane) * 128;
        for (int i = 0; i < 32; ++i) rr[i] = v[i], rr[32 + i] = u[i];
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        v[i] += u[i];
        v[i] += __shfl_xor_sync(0xffffffffu, v[i], 16);
      }
    } else {
      float w2[32], w3[32];
      tmem_ld32(lane_base, v);
      tmem_ld32(lane_base + 32, u);
      tmem_ld32(lane_base + 64, w2);
      tmem_ld32(lane_base + 96, w3);
      if constexpr (DUMP) {
        float* rr = raw + (static_cast<size_t>(blockIdx.x) * n_items + it) * 128 * 128 + (32 * wid + lane) * 128;
        for (int i = 0; i < 32; ++i) rr[i] = v[i], rr[32 + i] = u[i], rr[64 + i] = w2[i], rr[96 + i] = w3[i];
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = (v[i] + u[i]) + (w2[i] + w3[i]);
    }
    if (lane < 16) {
      float* o = out + ((static_cast<size_t>(blockIdx.x) * n_items + it) * 64 + 16 * wid + lane) * 32;
#pragma unroll
      for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
  }
  if (wid == 0) tmem_free<COLS>(tbase);
}

// ---- host ----------------------------------------------------------------
static float bf16_rn(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  const uint32_t r = u + 0x7fffu + ((u >> 16) & 1u);
  const uint32_t h = r & 0xffff0000u;
  float o;
  memcpy(&o, &h, 4);
  return o;
}

template <bool ILV>
static int check(const std::vector<float>& U1, const std::vector<float>& U2, const float* dU1, const float* dU2, int rows,
                 int R, int item_picks, const char* what) {
  const int n_items = 2, ppw = n_items * item_picks, ctas = 2;
  std::vector<Pick> picks(static_cast<size_t>(ctas) * 4 * ppw);
  uint64_t s = 88172645463325252ull;
  auto rnd = [&]() {
    s ^= s << 13, s ^= s >> 7, s ^= s << 17;
    return s;
  };
  for (auto& p : picks) p = {static_cast<uint32_t>(rnd() % rows), static_cast<uint32_t>(rnd() % rows),
                             static_cast<float>((rnd() % 1000) / 200.0), 0u};
  Pick* dp;
  float *dout, *draw;
  CK(cudaMalloc(&dp, picks.size() * sizeof(Pick)));
  CK(cudaMemcpy(dp, picks.data(), picks.size() * sizeof(Pick), cudaMemcpyHostToDevice));
  const size_t no = static_cast<size_t>(ctas) * n_items * 64 * 32, nr = static_cast<size_t>(ctas) * n_items * 128 * 128;
  CK(cudaMalloc(&dout, no * 4));
  CK(cudaMalloc(&draw, nr * 4));
  CK(cudaMemset(draw, 0, nr * 4));
  const int smem = 4 * NT * kTileBytes + 4 * RING * 16 + 4 * (NT + 1) * 8 + 16;
  CK(cudaFuncSetAttribute(k_gram<ILV, true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_gram<ILV, true, 3><<<ctas, 128, smem>>>(dU1, dU2, dp, ppw, item_picks, R, dout, draw, 0);
  CK(cudaDeviceSynchronize());
  std::vector<float> out(no), raw(nr);
  CK(cudaMemcpy(out.data(), dout, no * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(raw.data(), draw, nr * 4, cudaMemcpyDeviceToHost));
  double worst = 0, worst_h = 0, bias = 0;
  size_t nb = 0;
  for (int c = 0; c < ctas; ++c)
    for (int it = 0; it < n_items; ++it) {
      std::vector<double> D(64 * 32, 0.0), H(32 * 32, 0.0);
      for (int w = 0; w < 4; ++w)
        for (int e = 0; e < item_picks; ++e) {
          const Pick& p = picks[(static_cast<size_t>(c) * 4 + w) * ppw + static_cast<size_t>(it) * item_picks + e];
          float k[32], hi[32], lo[32];
          for (int f = 0; f < 32; ++f) {
            k[f] = f < R ? U1[static_cast<size_t>(p.j) * 32 + f] * U2[static_cast<size_t>(p.k) * 32 + f] : f == R ? p.x : 0.f;
            hi[f] = bf16_rn(k[f]);
            lo[f] = bf16_rn(k[f] - hi[f]);
          }
          for (int a = 0; a < 32; ++a)
            for (int b = 0; b < 32; ++b) {
              D[a * 32 + b] += static_cast<double>(hi[a]) * hi[b];
              D[(32 + a) * 32 + b] += static_cast<double>(lo[a]) * hi[b];
              H[a * 32 + b] += static_cast<double>(k[a]) * k[b];
            }
        }
      const float* o = out.data() + (static_cast<size_t>(c) * n_items + it) * 64 * 32;
      double dmax = 0;
      for (int i = 0; i < 64 * 32; ++i) dmax = std::max(dmax, std::fabs(D[i]));
      for (int i = 0; i < 64 * 32; ++i) {
        worst = std::max(worst, std::fabs(o[i] - D[i]) / dmax);
        if (i < 32 * 32 && D[i] > 0.01 * dmax) bias += (o[i] - D[i]) / D[i], ++nb;
      }
      for (int a = 0; a <= R; ++a)
        for (int b = 0; b <= R; ++b) {
          const double h = static_cast<double>(o[a * 32 + b]) + o[(32 + a) * 32 + b] + o[(32 + b) * 32 + a];
          worst_h = std::max(worst_h, std::fabs(h - H[a * 32 + b]) / std::fabs(H[a * 32 + b] + 1e-30));
        }
    }
  printf("%s: ILV %d R %d item_picks/warp %d : D max err / max|D| %.3e ; H rel err (hi/lo scheme) %.3e ; mean signed rel err of hi.hi %.3e\n",
         what, int(ILV), R, item_picks, worst, worst_h, nb ? bias / nb : 0.0);
  if (worst > 1e-4) {  // layout wrong: show where the numbers landed
    int shown = 0;
    for (int l = 0; l < 128 && shown < 12; ++l)
      for (int cidx = 0; cidx < 128 && shown < 12; ++cidx)
        if (raw[l * 128 + cidx] != 0.f) printf("  raw[lane %d][col %d] = %g\n", l, cidx, raw[l * 128 + cidx]), ++shown;
  }
  cudaFree(dp), cudaFree(dout), cudaFree(draw);
  return worst <= 1e-4 ? 0 : 1;
}

template <bool ILV, int STAGES, int NO = 2>
static void bench(const float* dU1, const float* dU2, int rows, int R, int ctas_per_sm, int pad_kb, int sms) {
  const int item_picks = 256, n_items = 64, ppw = item_picks * n_items;
  const int ctas = sms * ctas_per_sm;
  const size_t np = static_cast<size_t>(ctas) * 4 * ppw;
  std::vector<Pick> picks(np);
  uint64_t s = 0x9e3779b97f4a7c15ull;
  auto rnd = [&]() {
    s ^= s << 13, s ^= s >> 7, s ^= s << 17;
    return s;
  };
  for (auto& p : picks) p = {static_cast<uint32_t>(rnd() % rows), static_cast<uint32_t>(rnd() % rows), 1.5f, static_cast<uint32_t>(rnd() % 1000)};
  Pick* dp;
  float* dout;
  CK(cudaMalloc(&dp, np * sizeof(Pick)));
  CK(cudaMemcpy(dp, picks.data(), np * sizeof(Pick), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dout, static_cast<size_t>(ctas) * n_items * 64 * 32 * 4));
  const int smem = 4 * NT * kTileBytes + 4 * RING * 16 + 4 * (NT + 1) * 8 + 16 + pad_kb * 1024;
  CK(cudaFuncSetAttribute(k_gram<ILV, false, STAGES, NO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gram<ILV, false, STAGES, NO>, 128, smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  float best = 1e9f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k_gram<ILV, false, STAGES, NO><<<ctas, 128, smem>>>(dU1, dU2, dp, ppw, item_picks, R, dout, nullptr, 0);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best = std::min(best, ms);
  }
  printf("bench NO %d ILV %d STAGES %d R %d: %d CTAs/SM x 4 warps (occupancy %d), smem %d KB/CTA: %.3f ms, %.1f G picks/s\n", NO, int(ILV), STAGES, R,
         ctas_per_sm, occ, smem / 1024, best, np / best * 1e-6);
  cudaFree(dp), cudaFree(dout);
}

int main(int argc, char** argv) {
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, 0));
  const int rows = argc > 3 ? atoi(argv[3]) : 10000;  // factor rows (256: L1-resident gathers)
  std::vector<float> U1(static_cast<size_t>(rows) * 32), U2(U1.size());
  uint64_t s = 12345;
  auto rnd = [&]() {
    s ^= s << 13, s ^= s >> 7, s ^= s << 17;
    return static_cast<float>((s >> 40) * (1.0 / 16777216.0));
  };
  for (auto& v : U1) v = rnd();
  for (auto& v : U2) v = rnd();
  float *dU1, *dU2;
  CK(cudaMalloc(&dU1, U1.size() * 4));
  CK(cudaMalloc(&dU2, U2.size() * 4));
  CK(cudaMemcpy(dU1, U1.data(), U1.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dU2, U2.data(), U2.size() * 4, cudaMemcpyHostToDevice));
  if (argc > 2) {  // one configuration (for ncu): umma_gram <stages> <ctas per SM>
    if (atoi(argv[1]) == 3) bench<true, 3>(dU1, dU2, rows, 20, atoi(argv[2]), 0, pr.multiProcessorCount);
    else bench<true, 2>(dU1, dU2, rows, 20, atoi(argv[2]), 0, pr.multiProcessorCount);
    return 0;
  }
  int bad = 0;
  bad += check<false>(U1, U2, dU1, dU2, rows, 20, 16, "one tile");
  bad += check<false>(U1, U2, dU1, dU2, rows, 20, 100, "partial tiles");
  bad += check<true>(U1, U2, dU1, dU2, rows, 20, 16, "one tile");
  bad += check<true>(U1, U2, dU1, dU2, rows, 20, 100, "partial tiles");
  bad += check<true>(U1, U2, dU1, dU2, rows, 31, 250, "rank 31");
  bad += check<true>(U1, U2, dU1, dU2, rows, 20, 256, "item of 1024 picks");
  bad += check<true>(U1, U2, dU1, dU2, rows, 20, 4096, "item of 16384 picks (bias)");
  printf("checks failed: %d\n", bad);
  if (argc > 1 && !strcmp(argv[1], "check")) return bad;  // correctness part only (tests/test_microbench_umma.py)
  const int sms = pr.multiProcessorCount;
  for (int cps : {2, 3, 4}) bench<true, 2>(dU1, dU2, rows, 20, cps, 0, sms);
  for (int cps : {2, 3, 4}) bench<true, 3>(dU1, dU2, rows, 20, cps, 0, sms);
  bench<true, 3>(dU1, dU2, rows, 31, 3, 0, sms);
  for (int cps : {2, 3, 4}) bench<true, 2, 3>(dU1, dU2, rows, 31, cps, 0, sms);
  for (int cps : {2, 3}) bench<true, 3, 3>(dU1, dU2, rows, 31, cps, 0, sms);
  bench<true, 3>(dU1, dU2, rows, 20, 3, 24, sms);
  bench<true, 2>(dU1, dU2, rows, 20, 4, 24, sms);
  return bad;
}
