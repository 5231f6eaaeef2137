#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
// Hybrid gather microbenchmark: per pick two factor rows (ld 24, L2-resident),
// mode 1 by LDG in the pair (fragment) layout, mode 2 either by LDG too
// (baseline) or by TMA tile::gather4 into a per-warp stage ring read back
// with LDS in the same pair layout.  Reports G picks/s.
template <int ST>
struct Ring { float buf[ST][8][24]; uint64_t bar[ST]; };
__device__ __forceinline__ uint32_t sptr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(256, 2) k_ldg2(const float* __restrict__ U1, const float* __restrict__ U2,
                                                 const uint32_t* __restrict__ i1, const uint32_t* __restrict__ i2,
                                                 int groups, float* out) {
  extern __shared__ float sm[];
  if (groups < 0) sm[threadIdx.x] = 0;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float acc = 0.f;
  const uint32_t* a = i1 + (size_t)warp * groups * 8;
  const uint32_t* b = i2 + (size_t)warp * groups * 8;
  for (int it = 0; it < groups; ++it) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float* p1 = U1 + (size_t)a[it * 8 + 2 * t + q] * 24;
      const float* p2 = U2 + (size_t)b[it * 8 + 2 * t + q] * 24;
      float2 v1 = __ldg(reinterpret_cast<const float2*>(p1 + 2 * g));
      float w1 = __ldg(p1 + 16 + g);
      float2 v2 = __ldg(reinterpret_cast<const float2*>(p2 + 2 * g));
      float w2 = __ldg(p2 + 16 + g);
      acc += v1.x * v2.x + v1.y * v2.y + w1 * w2;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

template <int ST>
__global__ void __launch_bounds__(256, 2) k_hybrid(const __grid_constant__ CUtensorMap tm, const float* __restrict__ U1,
                                                   const uint32_t* __restrict__ i1, const uint32_t* __restrict__ i2,
                                                   int groups, float* out) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  Ring<ST>* ring = reinterpret_cast<Ring<ST>*>(smraw + wid * ((sizeof(Ring<ST>) + 127) / 128 * 128));
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t* a = i1 + (size_t)warp * groups * 8;
  const uint32_t* b = i2 + (size_t)warp * groups * 8;
  if (lane == 0)
    for (int s = 0; s < ST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sptr(&ring->bar[s])));
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  auto issue = [&](int it, int s) {
    if (lane == 0) {
      const uint32_t* r = b + it * 8;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(&ring->bar[s])), "r"(8 * 96) : "memory");
      for (int h = 0; h < 2; ++h)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(sptr(&ring->buf[s][4 * h][0])), "l"(&tm), "r"(0), "r"(r[4 * h]), "r"(r[4 * h + 1]), "r"(r[4 * h + 2]), "r"(r[4 * h + 3]),
            "r"(sptr(&ring->bar[s])) : "memory");
    }
  };
  for (int s = 0; s < ST && s < groups; ++s) issue(s, s);
  float acc = 0.f;
  uint32_t phase = 0;
  for (int it = 0; it < groups; ++it) {
    const int s = it % ST;
    // mode 1 by LDG first (in flight while waiting for the TMA stage)
    float2 v1[2];
    float w1[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float* p1 = U1 + (size_t)a[it * 8 + 2 * t + q] * 24;
      v1[q] = __ldg(reinterpret_cast<const float2*>(p1 + 2 * g));
      w1[q] = __ldg(p1 + 16 + g);
    }
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(sptr(&ring->bar[s])), "r"((phase >> s) & 1u) : "memory");
    phase ^= 1u << s;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float* p2 = &ring->buf[s][2 * t + q][0];
      const float2 v2 = *reinterpret_cast<const float2*>(p2 + 2 * g);
      const float w2 = p2[16 + g];
      acc += v1[q].x * v2.x + v1[q].y * v2.y + w1[q] * w2;
    }
    __syncwarp();
    if (it + ST < groups) issue(it + ST, s);
  }
  if (acc == 12345.f) out[0] = acc;
}

// LDG pair both modes with L1 no-allocate (.cg) loads
__global__ void __launch_bounds__(256, 2) k_ldg2cg(const float* __restrict__ U1, const float* __restrict__ U2,
                                                   const uint32_t* __restrict__ i1, const uint32_t* __restrict__ i2,
                                                   int groups, float* out) {
  extern __shared__ float sm[];
  if (groups < 0) sm[threadIdx.x] = 0;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float acc = 0.f;
  const uint32_t* a = i1 + (size_t)warp * groups * 8;
  const uint32_t* b = i2 + (size_t)warp * groups * 8;
  for (int it = 0; it < groups; ++it) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float* p1 = U1 + (size_t)a[it * 8 + 2 * t + q] * 24;
      const float* p2 = U2 + (size_t)b[it * 8 + 2 * t + q] * 24;
      float2 v1 = __ldcg(reinterpret_cast<const float2*>(p1 + 2 * g));
      float w1 = __ldcg(p1 + 16 + g);
      float2 v2 = __ldcg(reinterpret_cast<const float2*>(p2 + 2 * g));
      float w2 = __ldcg(p2 + 16 + g);
      acc += v1.x * v2.x + v1.y * v2.y + w1 * w2;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

// mode 1 from a shared-memory factor tile (rows drawn inside the tile: the
// j-tiling idea), mode 2 by LDG pair
template <int J>
__global__ void __launch_bounds__(256, 2) k_tile(const float* __restrict__ U1, const float* __restrict__ U2,
                                                 const uint32_t* __restrict__ i1, const uint32_t* __restrict__ i2,
                                                 int groups, float* out) {
  extern __shared__ __align__(16) float tile[];  // [J][24]
  for (int q = threadIdx.x; q < J * 24; q += blockDim.x) tile[q] = U1[q];
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float acc = 0.f;
  const uint32_t* a = i1 + (size_t)warp * groups * 8;
  const uint32_t* b = i2 + (size_t)warp * groups * 8;
  for (int it = 0; it < groups; ++it) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float* p1 = tile + (a[it * 8 + 2 * t + q] % J) * 24;
      const float* p2 = U2 + (size_t)b[it * 8 + 2 * t + q] * 24;
      float2 v1 = *reinterpret_cast<const float2*>(p1 + 2 * g);
      float w1 = p1[16 + g];
      float2 v2 = __ldg(reinterpret_cast<const float2*>(p2 + 2 * g));
      float w2 = __ldg(p2 + 16 + g);
      acc += v1.x * v2.x + v1.y * v2.y + w1 * w2;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int rows = 10000, W = 296 * 8, groups = 2048;
  float *U1, *U2, *out; uint32_t *i1, *i2;
  cudaMalloc(&U1, sizeof(float) * rows * 24 + 4096);
  cudaMalloc(&U2, sizeof(float) * rows * 24 + 4096);
  cudaMemset(U1, 0, sizeof(float) * rows * 24);
  cudaMemset(U2, 0, sizeof(float) * rows * 24);
  size_t n = (size_t)W * groups * 8;
  cudaMalloc(&i1, n * 4); cudaMalloc(&i2, n * 4);
  uint32_t* h = new uint32_t[n];
  uint64_t s = 88172645463325252ull;
  for (size_t i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % rows; }
  cudaMemcpy(i1, h, n * 4, cudaMemcpyHostToDevice);
  for (size_t i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % rows; }
  cudaMemcpy(i2, h, n * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&out, 4);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {24, (cuuint64_t)rows}, strides[1] = {96};
  cuuint32_t box[2] = {24, 1}, es[2] = {1, 1};
  CUresult rc = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, U2, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)rc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, int smem, const char* name, auto... extra) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      kern<<<296, 256, smem>>>(extra..., i1, i2, groups, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("%-40s smem %6d  %.3f ms  %.2f G picks/s  (%s)\n", name, smem, ms, n / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int kb : {0, 16, 26, 36, 48, 60, 74, 100}) run(k_ldg2, kb * 1024, "LDG pair, both modes", U1, U2);
  for (int kb : {26, 74}) run(k_ldg2cg, kb * 1024, "LDG.cg pair, both modes", U1, U2);
  run(k_tile<512>, 512 * 96, "mode 1 from smem tile J=512", U1, U2);
  run(k_tile<1024>, 1024 * 96, "mode 1 from smem tile J=1024", U1, U2);
  run(k_hybrid<2>, 8 * 2 * 1024 + 8192, "hybrid ST=2 (mode 2 via TMA)", tm, U1);
  run(k_hybrid<4>, 8 * 4 * 1024, "hybrid ST=4", tm, U1);
  run(k_hybrid<6>, 8 * 6 * 1024, "hybrid ST=6", tm, U1);
  run(k_hybrid<8>, 8 * 8 * 1024, "hybrid ST=8", tm, U1);
  run(k_hybrid<8>, 96 * 1024, "hybrid ST=8 (96 KB carve-out)", tm, U1);
}
