#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
// Gather microbenchmark: each warp gathers groups of 8 random rows of a
// 10000 x LD float matrix (L2-resident) in different lane layouts.
template <int V, int LD>
__global__ void __launch_bounds__(256, 2) k(const float* __restrict__ U, const uint32_t* __restrict__ idx, int groups, float* out) {
  extern __shared__ float sm[];
  if (groups < 0) sm[threadIdx.x] = 0;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float acc = 0.f;
  const uint32_t* id = idx + (size_t)warp * groups * 8;
  for (int it = 0; it < groups; ++it) {
    const uint32_t* r = id + it * 8;
    if (V == 1) {  // pair: picks 2t, 2t+1; LDG.64 at 2g, LDG.32 at 16+g
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float* b = U + (size_t)r[2 * t + q] * LD;
        float2 v = __ldg(reinterpret_cast<const float2*>(b + 2 * g));
        float w = __ldg(b + 16 + g);
        acc += v.x * v.y + w;
      }
    } else if (V == 9) {  // pair on a row-rotated layout: rows with row % 4 == 1 (byte offset 96 mod 128) store
                          // features 16-23 first, so the 64-byte part never straddles an L1 line
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t row = r[2 * t + q];
        const float* b = U + (size_t)row * LD;
        const bool rot = (row & 3u) == 1u;
        float2 v = __ldg(reinterpret_cast<const float2*>(b + (rot ? 8 : 0) + 2 * g));
        float w = __ldg(b + (rot ? 0 : 16) + g);
        acc += v.x * v.y + w;
      }
    } else if (V == 2) {  // natural: 8 lanes per row, lanes g<6 float4
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float* b = U + (size_t)r[4 * h + (lane >> 3)] * LD;
        const int s = lane & 7;
        if (s < LD / 4) {
          float4 v = __ldg(reinterpret_cast<const float4*>(b) + s);
          acc += v.x * v.y + v.z * v.w;
        }
      }
    } else if (V == 3) {  // scalar: 3 x LDG.32 per pick pair lane (g, t)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float* b = U + (size_t)r[2 * t + q] * LD;
        acc += __ldg(b + g) + __ldg(b + g + 8) * __ldg(b + g + 16);
      }
    } else if (V == 5) {  // natural float4 (8 lanes per 128-byte row) + SHFL into the fragment layout
      float4 v[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float* b = U + (size_t)r[4 * h + (lane >> 3)] * LD;
        v[h] = __ldg(reinterpret_cast<const float4*>(b) + (lane & 7));
      }
      // lane (g,t) wants picks t and t+4, features 4g + f (f = 0..3): register f of lane 8t + g
      const int src = 8 * t + g;
      float f0 = __shfl_sync(0xffffffffu, v[0].x, src), f1 = __shfl_sync(0xffffffffu, v[0].y, src);
      float f2 = __shfl_sync(0xffffffffu, v[0].z, src), f3 = __shfl_sync(0xffffffffu, v[0].w, src);
      float e0 = __shfl_sync(0xffffffffu, v[1].x, src), e1 = __shfl_sync(0xffffffffu, v[1].y, src);
      float e2 = __shfl_sync(0xffffffffu, v[1].z, src), e3 = __shfl_sync(0xffffffffu, v[1].w, src);
      acc += f0 * f1 + f2 * f3 + e0 * e1 + e2 * e3;
    } else if (V == 6) {  // natural float4, no transposition (reference for V5)
      float4 v[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float* b = U + (size_t)r[4 * h + (lane >> 3)] * LD;
        v[h] = __ldg(reinterpret_cast<const float4*>(b) + (lane & 7));
      }
      acc += v[0].x * v[0].y + v[0].z * v[0].w + v[1].x * v[1].y + v[1].z * v[1].w;
    } else if (V == 7) {  // quad fragment layout: lane (g,t) reads picks 2t+q, float4 at 4g (8 strided lanes per row)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float* b = U + (size_t)r[2 * t + q] * LD;
        float4 v = __ldg(reinterpret_cast<const float4*>(b + 4 * g));
        acc += v.x * v.y + v.z * v.w;
      }
    } else if (V == 8) {  // quad, pick t + 4q (fragment k-index order)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float* b = U + (size_t)r[t + 4 * q] * LD;
        float4 v = __ldg(reinterpret_cast<const float4*>(b + 4 * g));
        acc += v.x * v.y + v.z * v.w;
      }
    } else if (V == 4) {  // natural float2: 12 lanes per row (2.67 rows per instr) -> 16 lanes per row, 2 rows per instr
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float* b = U + (size_t)r[2 * h + (lane >> 4)] * LD;
        const int s = lane & 15;
        if (s < LD / 2) {
          float2 v = __ldg(reinterpret_cast<const float2*>(b) + s);
          acc += v.x * v.y;
        }
      }
    }
  }
  if (acc == 12345.f) out[0] = acc;
}
int main() {
  const int rows = 10000, LD = 24, W = 296 * 8, groups = 4096;
  float* U; uint32_t* idx; float* out;
  cudaMalloc(&U, sizeof(float) * rows * 32 + 4096);
  cudaMemset(U, 0, sizeof(float) * rows * 32);
  size_t n = (size_t)W * groups * 8;
  cudaMalloc(&idx, n * 4);
  uint32_t* h = new uint32_t[n];
  uint64_t s = 88172645463325252ull;
  for (size_t i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % rows; }
  cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int smem = 0;
  auto run = [&](auto kern, const char* name) {
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kern<<<296, 256, smem>>>(U, idx, groups, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("%-28s %.3f ms  %.2f G rows/s\n", name, ms, n / (ms * 1e-3) / 1e9);
  };
  for (int sm_kb : {0, 74}) {
  smem = sm_kb * 1024;
  printf("smem per CTA %d KB\n", sm_kb);
  run(k<1, 24>, "pair ld24 (LDG.64+LDG.32)");
  run(k<9, 24>, "pair ld24, rotated rows (no straddle)");
  run(k<2, 24>, "natural ld24 float4");
  run(k<3, 24>, "scalar ld24 3xLDG.32");
  run(k<4, 24>, "natural ld24 float2");
  run(k<1, 32>, "pair ld32");
  run(k<2, 32>, "natural ld32 float4");
  run(k<5, 32>, "natural ld32 float4 + 8 SHFL");
  run(k<6, 32>, "natural ld32 float4 (V5 w/o SHFL)");
  run(k<7, 32>, "quad ld32 (lane g,t: pick 2t+q, float4 4g)");
  run(k<8, 32>, "quad ld32 (lane g,t: pick t+4q, float4 4g)");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
