// tcgen05 (5th-generation tensor core) helpers for sm_100a: tensor-memory
// allocation, shared-memory matrix descriptors, the single-thread MMA issue,
// completion through mbarriers and the accumulator read-back.  Raw PTX; no
// CUTLASS.  Used by
// tools/microbench/umma_gram.cu (the product does not use it: see
// profiles/r02_tcgen05_experiment.txt).
//
// Operand tile (one per 16 picks), MN-major with the 128-byte swizzle: a pick
// is one 128-byte row [hi(32 features) | lo(32 features)] of bf16, eight rows
// form a 1024-byte swizzle atom (16-byte chunk c of row r is stored at chunk
// position c ^ r), a tile is two atoms (2048 bytes, 1024-byte aligned).
//   A = the whole row      (M = 64: 32 hi features, then 32 lo features)
//   B = its first 64 bytes (N = 32: the hi features)
// so one tcgen05.mma (kind::f16, M 64, N 32, K 16) adds
//   D[64 x 32] += [hi; lo] hi^T   over the tile's 16 picks,
// and sum k k^T ~= D[i][j] + D[32 + i][j] + D[32 + j][i].
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace ntcb {
namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- tensor memory -------------------------------------------------------
// one full warp allocates `cols` (a power of two >= 32) columns; the base
// address lands in *slot (shared memory)
template <int COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)), "r"(COLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
template <int COLS>
__device__ __forceinline__ void tmem_free(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "r"(COLS) : "memory");
}
__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core's reads
__device__ __forceinline__ void fence_smem_to_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// ---- mbarrier ------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra D_%=;\n"
      "bra W_%=;\n"
      "D_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---- descriptors ---------------------------------------------------------
// shared-memory matrix descriptor of an MN-major, 128-byte-swizzled operand:
// start address (16-byte units), leading byte offset (between 64-element MN
// atoms; one atom here), stride byte offset 1024 (between 8-row K atoms),
// descriptor version 1 (sm_100), layout type 2 (SWIZZLE_128B)
__device__ __forceinline__ uint64_t smem_desc_mn_sw128(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3ffffu) >> 4) | (static_cast<uint64_t>(1024u >> 4) << 16) |
         (static_cast<uint64_t>(1024u >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: fp32 accumulate, bf16 x bf16, both operands
// MN-major, N at [17,23) in units of 8, M at [24,29) in units of 16
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] B[smem]; one thread issues for the CTA
__device__ __forceinline__ void mma_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// the mbarrier gets one arrival when every MMA issued so far by this thread
// has completed (implies tcgen05.fence::before_thread_sync)
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

// ---- accumulator read-back -------------------------------------------------
// warp w reads tensor-memory lanes 32 w .. 32 w + 31 (its sub-partition):
// thread t gets lane 32 w + t, 32 consecutive columns from `taddr`
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- operand tile ------------------------------------------------------------
constexpr int kTileBytes = 2048;  // 16 picks x 128 bytes
// byte offset, inside a tile, of 16-byte chunk `c` (0..7) of tile row `p` (0..15)
__device__ __forceinline__ uint32_t tile_chunk_off(int p, int c) {
  const int r = p & 7;
  return static_cast<uint32_t>((p >> 3) * 1024 + r * 128 + ((c ^ r) << 4));
}
// k (4 consecutive features, fp32) -> bf16 hi and lo = bf16(k - hi), packed
__device__ __forceinline__ void split_bf16(const float4& k, uint2& hi, uint2& lo) {
  __nv_bfloat162 h01 = __floats2bfloat162_rn(k.x, k.y);
  __nv_bfloat162 h23 = __floats2bfloat162_rn(k.z, k.w);
  const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
  __nv_bfloat162 l01 = __floats2bfloat162_rn(k.x - f01.x, k.y - f01.y);
  __nv_bfloat162 l23 = __floats2bfloat162_rn(k.z - f23.x, k.w - f23.y);
  hi.x = *reinterpret_cast<uint32_t*>(&h01);
  hi.y = *reinterpret_cast<uint32_t*>(&h23);
  lo.x = *reinterpret_cast<uint32_t*>(&l01);
  lo.y = *reinterpret_cast<uint32_t*>(&l23);
}
// lane q (0..7) of a pick's octet stores features 4q..4q+3: hi at logical
// byte 8q of the row, lo at 64 + 8q
__device__ __forceinline__ void tile_store(unsigned char* tile, int p, int q, const uint2& hi, const uint2& lo) {
  const uint32_t sub = static_cast<uint32_t>((q & 1) << 3);
  *reinterpret_cast<uint2*>(tile + tile_chunk_off(p, q >> 1) + sub) = hi;
  *reinterpret_cast<uint2*>(tile + tile_chunk_off(p, 4 + (q >> 1)) + sub) = lo;
}
// tile row handled by octet i (0..3) in step s (0..3): the two octets of a
// half-warp write rows r and r + 4, whose hi (and lo) halves sit in disjoint
// banks under the swizzle -- conflict-free 8-byte stores
__device__ __forceinline__ int tile_row_of(int s, int i) { return (s >> 1) * 8 + (s & 1) * 2 + (i >> 1) + 4 * (i & 1); }

}  // namespace umma
}  // namespace ntcb
