// Bit-exact mini-batch sampler: the reference's partial Fisher-Yates
// (nmc.cpp:44-63) over every slice of a mode view, one warp per slice,
// 32 draws resolved in parallel per step.
//
// Reference semantics for one slice of n entries, b = floor(c*n):
//   perm = iota(n); for j < b: r_j = j + next_below(n - j);
//   swap(perm[j], perm[r_j]); picks[j] = perm[j]
// with the row stream RngStream(rng).fork(l).fork(p) (nmc.cpp:236).
//
// Warp formulation.  Draw j only needs the stream counter, so lanes compute
// r_j for 32 consecutive j at once (state + (j+1)*G).  Lemire's product
// x * bound is formed from two 32x32->64 multiplies (bound < 2^31); a draw
// whose low 64-bit word falls below the bound might need the rejection loop
// of rng.hpp:36-43 -- then the whole chunk is replayed serially on lane 0,
// which is exact.  Within a chunk the swap chain is resolved without
// serialisation:
//   f(j)     = value at position j when step j runs
//            = f(link(j)) if an earlier lane of the chunk targeted position j
//              (link = last such lane), else perm[j] at chunk start;
//   picks[j] = f(prev(j)) if an earlier lane drew the same r (prev = last
//              such lane, via __match_any_sync), else perm[r_j] at chunk start;
// link chains are collapsed by pointer jumping over shuffles (5 rounds).
// After the chunk only positions >= chunk end can be read again, so only the
// last writer of each such position stores f.  perm lives in shared memory
// (u16 when n <= 65536, stored XOR position so that zero-fill == iota), or
// in a global per-entry scratch for slices larger than the smem budget.
//
// Output: one bit per view entry in `mask` (the sampled SET that the update
// kernel streams) and optionally the picks in draw order (parity tests).
#include "common.cuh"

namespace ntcb {

struct SampleArgs {
  const uint64_t* off;
  uint64_t row_begin, row_end;
  double c;
  uint64_t root;  // RngStream(rng).fork(l) raw state; row p uses fork(root, p)
  uint32_t* mask;
  unsigned long long* counters;  // [1] error key (early exit)
  uint32_t* dbg_picks;           // optional, picks in draw order
  const uint64_t* dbg_off;       // dbg offsets per row (relative to row_begin)
  uint32_t* gscratch;            // per-entry u32 scratch (indexed by view entry)
  uint64_t cap;                  // max slice length handled in shared memory
  uint32_t perm_bytes;           // per-warp smem bytes for perm
  uint32_t mask_bytes;           // per-warp smem bytes for the slice bitmask
  uint32_t warp_bytes;           // per-warp total
  int direct;                    // 1: `root` is the row stream itself (sample_row)
};

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSampleWarps = 2;

template <typename QT, bool SMASK>
__device__ __forceinline__ void fy_slice(QT* perm, uint32_t n, uint32_t b, uint64_t state,
                                         int lane, int* tgt, uint32_t* rtmp, uint32_t* smask,
                                         uint32_t* gmask, uint64_t beg, uint32_t* dbg) {
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t moff = SMASK ? static_cast<uint32_t>(beg & 31u) : 0u;
  const uint64_t lane_off = static_cast<uint64_t>(lane + 1) * kGolden;
  for (uint32_t j0 = 0; j0 < b; j0 += 32) {
    const uint32_t rem = b - j0;
    const uint32_t nvalid = rem < 32u ? rem : 32u;
    const bool act = static_cast<uint32_t>(lane) < nvalid;
    const uint32_t j = j0 + lane;
    const uint32_t bound = act ? n - j : 1u;
    const uint64_t x = mix64(state + lane_off);
    // 96-bit x*bound = (u << 32) + lo32(t)
    const uint64_t t = static_cast<uint64_t>(static_cast<uint32_t>(x)) * bound;
    const uint64_t u = static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * bound + (t >> 32);
    const bool maybe_reject = act && static_cast<uint32_t>(u) == 0u && static_cast<uint32_t>(t) < bound;
    uint32_t r;
    if (__ballot_sync(kFull, maybe_reject)) {
      // lo64 < bound somewhere: replay the chunk exactly (rng.hpp:32-45).
      uint64_t s = state;
      if (lane == 0) {
        for (uint32_t q = 0; q < nvalid; ++q) {
          const uint64_t bd = n - (j0 + q);
          s += kGolden;
          uint64_t xx = mix64(s);
          uint64_t l2 = xx * bd, h2 = __umul64hi(xx, bd);
          if (l2 < bd) {
            const uint64_t th = (0 - bd) % bd;
            while (l2 < th) {
              s += kGolden;
              xx = mix64(s);
              l2 = xx * bd;
              h2 = __umul64hi(xx, bd);
            }
          }
          rtmp[q] = static_cast<uint32_t>(j0 + q + h2);
        }
      }
      __syncwarp();
      r = act ? rtmp[lane] : 0u;
      state = __shfl_sync(kFull, s, 0);
      __syncwarp();
    } else {
      r = j + static_cast<uint32_t>(u >> 32);
      state += static_cast<uint64_t>(nvalid) * kGolden;
    }
    uint32_t aval = 0, cval = 0;
    if (act) {
      aval = (static_cast<uint32_t>(perm[j]) ^ j) & (sizeof(QT) == 2 ? 0xffffu : 0xffffffffu);
      cval = (static_cast<uint32_t>(perm[r]) ^ r) & (sizeof(QT) == 2 ? 0xffffu : 0xffffffffu);
    }
    uint32_t f = aval;
    const bool tg = act && r > j && r < j0 + 32u;
    if (__ballot_sync(kFull, tg)) {
      tgt[lane] = -1;
      __syncwarp();
      if (tg) atomicMax(&tgt[r - j0], lane);
      __syncwarp();
      int ptr = act ? tgt[lane] : -1;
#pragma unroll
      for (int it = 0; it < 5; ++it) {
        const int src = ptr < 0 ? lane : ptr;
        const uint32_t fv = __shfl_sync(kFull, f, src);
        const int pv = __shfl_sync(kFull, ptr, src);
        if (ptr >= 0) {
          f = fv;
          ptr = pv;
        }
      }
    }
    // slices are < 2^31 entries, so inactive lanes' keys never collide
    const uint32_t key = act ? r : (0x80000000u | static_cast<uint32_t>(lane));
    const uint32_t m = __match_any_sync(kFull, key);
    const uint32_t prev = m & lt;
    const int src = prev ? 31 - __clz(prev) : lane;
    const uint32_t fsrc = __shfl_sync(kFull, f, src);
    const uint32_t pick = prev ? fsrc : cval;
    const bool last_writer = act && (31 - __clz(m)) == lane;
    __syncwarp();
    if (last_writer && r >= j0 + 32u) perm[r] = static_cast<QT>(f ^ r);
    if (act) {
      if (SMASK) {
        const uint32_t lb = moff + pick;
        atomicOr(&smask[lb >> 5], 1u << (lb & 31u));
      } else {
        const uint64_t gb = beg + pick;
        atomicOr(&gmask[gb >> 5], 1u << (gb & 31u));
      }
      if (dbg) dbg[j] = pick;
    }
    __syncwarp();
  }
}

template <typename QT>
__global__ void __launch_bounds__(kSampleWarps * 32) k_sample(SampleArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* wbase = smem + static_cast<size_t>(wib) * a.warp_bytes;
  QT* sperm = reinterpret_cast<QT*>(wbase);
  uint32_t* smask = reinterpret_cast<uint32_t*>(wbase + a.perm_bytes);
  int* tgt = reinterpret_cast<int*>(wbase + a.perm_bytes + a.mask_bytes);
  uint32_t* rtmp = reinterpret_cast<uint32_t*>(tgt + 32);

  if (*reinterpret_cast<volatile unsigned long long*>(&a.counters[1]) != ~0ull) return;

  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kSampleWarps;
  for (uint64_t p = a.row_begin + blockIdx.x * kSampleWarps + wib; p < a.row_end; p += nw) {
    const uint64_t beg = a.off[p];
    const uint32_t n = static_cast<uint32_t>(a.off[p + 1] - beg);
    const uint32_t b = static_cast<uint32_t>(blocksize_for(a.c, n));
    if (b == 0) continue;  // row skipped (nmc.cpp:237)
    uint32_t* dbg = a.dbg_picks ? a.dbg_picks + a.dbg_off[p - a.row_begin] : nullptr;
    if (a.c >= 1.0) {  // slice order, no randomness (nmc.cpp:52-55); the update kernel
      if (dbg)         // then ignores the mask entirely.
        for (uint32_t t = lane; t < n; t += 32) dbg[t] = t;
      continue;
    }
    const uint64_t state = a.direct ? a.root : fork64(a.root, p);
    if (n <= a.cap) {
      // zero-fill == identity permutation in the XOR representation
      const uint32_t pw = static_cast<uint32_t>((n * sizeof(QT) + 15) / 16);
      uint4* p4 = reinterpret_cast<uint4*>(sperm);
      for (uint32_t w = lane; w < pw; w += 32) p4[w] = make_uint4(0, 0, 0, 0);
      const uint32_t nwords = static_cast<uint32_t>(((beg & 31u) + n + 31) / 32);
      for (uint32_t w = lane; w < nwords; w += 32) smask[w] = 0;
      __syncwarp();
      fy_slice<QT, true>(sperm, n, b, state, lane, tgt, rtmp, smask, nullptr, beg, dbg);
      __syncwarp();
      uint32_t* g = a.mask + (beg >> 5);
      const uint32_t last = nwords - 1;
      for (uint32_t w = lane; w < nwords; w += 32) {
        const uint32_t v = smask[w];
        // interior words belong to this slice alone; boundary words are shared
        if (w != 0 && w != last)
          g[w] = v;
        else if (v)
          atomicOr(&g[w], v);
      }
      __syncwarp();
    } else {
      uint32_t* gp = a.gscratch + beg;
      for (uint32_t t = lane; t < n; t += 32) gp[t] = 0;
      __syncwarp();
      fy_slice<uint32_t, false>(gp, n, b, state, lane, tgt, rtmp, nullptr, a.mask, beg, dbg);
      __syncwarp();
    }
  }
}

// Host launcher.  Returns the number of kernel launches issued.
int launch_sample(ntcb_context* ctx, cudaStream_t stream, uint32_t* mask, int mode,
                  uint64_t row_begin, uint64_t row_end, double c, uint64_t root,
                  uint32_t* dbg_picks, const uint64_t* dbg_off, int direct) {
  const DeviceView& v = ctx->views[mode];
  if (row_end <= row_begin) return 0;
  if (v.max_slice >= (1ull << 31))
    fail(NTCB_EINVAL, "sampler: slices of 2^31 or more entries are not supported");
  SampleArgs a{};
  a.off = v.off;
  a.row_begin = row_begin;
  a.row_end = row_end;
  a.c = c;
  a.root = root;
  a.mask = mask;
  a.counters = ctx->counters;
  a.dbg_picks = dbg_picks;
  a.dbg_off = dbg_off;
  a.gscratch = ctx->perm_scratch;
  a.direct = direct;

  // Shared memory per warp: perm sized to the largest slice (u16 when the
  // values fit) plus the slice bitmask, up to ~56 KB; longer slices use the
  // global scratch.
  const uint64_t maxn = v.max_slice;
  const bool small = maxn <= 65536;
  const uint64_t esz = small ? 2 : 4;
  const uint64_t budget = 56 * 1024;
  uint64_t cap = maxn;
  if (cap * esz + cap / 8 + 512 > budget) cap = (budget - 512) * 8 / (8 * esz + 1);
  if (cap < 32) cap = 32;
  a.cap = cap;
  a.perm_bytes = static_cast<uint32_t>((cap * esz + 15) / 16 * 16);
  a.mask_bytes = static_cast<uint32_t>(((cap + 31) / 32 + 2) * 4 + 15) / 16 * 16;
  a.warp_bytes = a.perm_bytes + a.mask_bytes + 64 * 4;
  const size_t smem = static_cast<size_t>(a.warp_bytes) * kSampleWarps;
  if (maxn > cap && ctx->perm_scratch == nullptr)
    fail(NTCB_ECUDA, "sampler: slice exceeds shared-memory budget and no scratch allocated");

  const uint64_t rows = row_end - row_begin;
  int per_sm = 0;
  if (small) {
    NTCB_CUDA(cudaFuncSetAttribute(k_sample<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    NTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sample<uint16_t>,
                                                            kSampleWarps * 32, smem));
  } else {
    NTCB_CUDA(cudaFuncSetAttribute(k_sample<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    NTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sample<uint32_t>,
                                                            kSampleWarps * 32, smem));
  }
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (rows + kSampleWarps - 1) / kSampleWarps;
  const uint64_t cap_grid = static_cast<uint64_t>(per_sm) * ctx->sm_count;
  if (grid > cap_grid) grid = cap_grid;
  if (small)
    k_sample<uint16_t><<<static_cast<unsigned>(grid), kSampleWarps * 32, smem, stream>>>(a);
  else
    k_sample<uint32_t><<<static_cast<unsigned>(grid), kSampleWarps * 32, smem, stream>>>(a);
  NTCB_CUDA(cudaGetLastError());
  return 1;
}

}  // namespace ntcb
