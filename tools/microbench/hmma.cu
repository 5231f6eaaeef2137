#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_tf32(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 1, b1 = a0 ^ 2;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_bf16(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 1, b1 = a0 ^ 2;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(float* out, int iters) {
  float c[16]; for (int j = 0; j < 16; ++j) c[j] = threadIdx.x * j;
  float x = threadIdx.x * 0.5f, y = 1.0001f;
  for (int i = 0; i < iters * 8; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = fmaf(c[j], y, x);
  }
  float s = 0; for (int j = 0; j < 16; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    for (int w = 0; w < 3; ++w) {
      float ms;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (w == 0) k_tf32<<<148 * 2, warps * 16>>>(out, iters);
        else if (w == 1) k_bf16<<<148 * 2, warps * 16>>>(out, iters);
        else k_ffma<<<148 * 2, warps * 16>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      double nwarps = 148.0 * 2 * warps / 2;
      if (w < 2) {
        double mmas = nwarps * iters * 8;
        double flop = mmas * (w == 0 ? 16 * 8 * 8 * 2 : 16 * 8 * 16 * 2);
        printf("%s warps/SM=%d: %.3f ms, %.2f mma/clk/SM (1.965GHz), %.1f TFLOP/s\n", w == 0 ? "tf32" : "bf16", warps, ms,
               mmas / (ms * 1e-3) / 148 / 1.965e9, flop / (ms * 1e-3) / 1e12);
      } else {
        double ffma = nwarps * 32 * iters * 8 * 16;
        printf("ffma warps/SM=%d: %.3f ms, %.1f TFLOP/s\n", warps, ms, 2 * ffma / (ms * 1e-3) / 1e12);
      }
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
