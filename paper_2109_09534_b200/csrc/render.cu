// Dense CPD evaluation of an H x W x 3 model into 8-bit pixels: the
// reference's render_model (image.cpp:161-183, the image-completion demo of
// the paper's section IV.A), SURVEY.md §8f row 4.
//
// pixel (i, j, ch) = quantize(sum_r U1(i, r) U2(j, r) U3(ch, r)),
// quantize(v) = lround(min(255, max(0, v))) (image.cpp:47-50).  The sum runs
// in fp64 over the resident fp32 factors with the reference's association
// ((U1 U2) U3, r ascending) and explicitly rounded operations (no FMA
// contraction), so fp32-representable factors give the reference's pixels
// bit for bit.  HBM/launch bound: one thread per pixel, the rank-R rows of
// U1 and U2 read through L1/L2, U3 (3 x R) in shared memory.
#include <algorithm>

#include "common.cuh"

namespace ntcb {

namespace {

__global__ void k_render(const float* __restrict__ U1, const float* __restrict__ U2,
                         const float* __restrict__ U3, uint64_t H, uint64_t W, int R, int ld,
                         uint8_t* __restrict__ out) {
  extern __shared__ double u3[];  // [3][R]
  for (int q = threadIdx.x; q < 3 * R; q += blockDim.x) u3[q] = static_cast<double>(U3[(q / R) * ld + q % R]);
  __syncthreads();
  const uint64_t n = H * W;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = p / W, j = p - i * W;
    const float* a = U1 + i * ld;
    const float* b = U2 + j * ld;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int r = 0; r < R; ++r) {
      const double ab = __dmul_rn(static_cast<double>(__ldg(a + r)), static_cast<double>(__ldg(b + r)));
      v0 = __dadd_rn(v0, __dmul_rn(ab, u3[r]));
      v1 = __dadd_rn(v1, __dmul_rn(ab, u3[R + r]));
      v2 = __dadd_rn(v2, __dmul_rn(ab, u3[2 * R + r]));
    }
    const double v[3] = {v0, v1, v2};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const double c = fmin(255.0, fmax(0.0, v[ch]));
      out[3 * p + ch] = static_cast<uint8_t>(llround(c));
    }
  }
}

}  // namespace

void render_model(ntcb_context* ctx, uint8_t* d_pixels) {
  const uint64_t H = ctx->dims[0], W = ctx->dims[1];
  const uint64_t n = H * W;
  if (!n) return;
  const int R = static_cast<int>(ctx->rank);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 16ull * ctx->sm_count));
  k_render<<<grid, 256, sizeof(double) * 3 * R, ctx->stream>>>(ctx->A[0], ctx->A[1], ctx->A[2], H, W, R,
                                                               static_cast<int>(ctx->ld), d_pixels);
  NTCB_CUDA(cudaGetLastError());
}

}  // namespace ntcb
