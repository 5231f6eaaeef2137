#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
// TMA gather4 vs LDG gathers of random 96-byte rows (10000 x 24 floats, L2-resident).
constexpr int ST = 4;  // stages per warp
__device__ __forceinline__ uint32_t sptr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void __launch_bounds__(256, 2) k_tma(const __grid_constant__ CUtensorMap tm, const uint32_t* __restrict__ idx, int groups, float* out) {
  extern __shared__ __align__(128) float sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  float* buf = sm + wid * (ST * 8 * 24 + 32);          // [ST][8][24]
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + ST * 8 * 24);  // [ST]
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t* id = idx + (size_t)warp * groups * 8;
  if (lane == 0)
    for (int s = 0; s < ST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sptr(bar + s)));
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  auto issue = [&](int it, int s) {
    if (lane == 0) {
      const uint32_t* r = id + it * 8;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(bar + s)), "r"(8 * 96) : "memory");
      for (int h = 0; h < 2; ++h)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(sptr(buf + (s * 8 + 4 * h) * 24)), "l"(&tm), "r"(0), "r"(r[4 * h]), "r"(r[4 * h + 1]), "r"(r[4 * h + 2]), "r"(r[4 * h + 3]),
            "r"(sptr(bar + s)) : "memory");
    }
  };
  for (int s = 0; s < ST && s < groups; ++s) issue(s, s);
  float acc = 0.f;
  uint32_t phase = 0;
  for (int it = 0; it < groups; ++it) {
    const int s = it % ST;
    // wait
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(sptr(bar + s)), "r"((phase >> s) & 1u) : "memory");
    phase ^= 1u << s;
    const float* b = buf + s * 8 * 24;
    const float* p0 = b + t * 24, *p1 = b + (t + 4) * 24;
    acc += p0[g] * p0[g + 8] + p0[g + 16] + p1[g] * p1[g + 8] + p1[g + 16];
    __syncwarp();
    if (it + ST < groups) issue(it + ST, s);
  }
  if (acc == 12345.f) out[0] = acc;
}
__global__ void __launch_bounds__(256, 2) k_ldg(const float* __restrict__ U, const uint32_t* __restrict__ idx, int groups, float* out) {
  extern __shared__ float sm[];
  if (groups < 0) sm[threadIdx.x] = 0;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float acc = 0.f;
  const uint32_t* id = idx + (size_t)warp * groups * 8;
  for (int it = 0; it < groups; ++it) {
    const uint32_t* r = id + it * 8;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float* b = U + (size_t)r[2 * t + q] * 24;
      float2 v = __ldg(reinterpret_cast<const float2*>(b + 2 * g));
      float w = __ldg(b + 16 + g);
      acc += v.x * v.y + w;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int rows = 10000, W = 296 * 8, groups = 4096;
  float* U; uint32_t* idx; float* out;
  cudaMalloc(&U, sizeof(float) * rows * 24 + 4096);
  cudaMemset(U, 0, sizeof(float) * rows * 24);
  size_t n = (size_t)W * groups * 8;
  cudaMalloc(&idx, n * 4);
  uint32_t* h = new uint32_t[n];
  uint64_t s = 88172645463325252ull;
  for (size_t i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % rows; }
  cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&out, 4);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {24, (cuuint64_t)rows}, strides[1] = {96};
  cuuint32_t box[2] = {24, 1}, es[2] = {1, 1};
  CUresult rc = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, U, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)rc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int smem = 74 * 1024;
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(e0); k_ldg<<<296, 256, smem>>>(U, idx, groups, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("ldg pair  %.3f ms %.1f G rows/s\n", ms, n / (ms * 1e-3) / 1e9);
    cudaEventRecord(e0); k_tma<<<296, 256, smem>>>(tm, idx, groups, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("tma g4    %.3f ms %.1f G rows/s\n", ms, n / (ms * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
