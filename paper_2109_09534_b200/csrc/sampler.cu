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
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <vector>

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
  uint32_t tiny_cap;             // slices up to this length are left to k_sample_tiny (0: none)
  uint32_t scan_w;               // k_sample_set: consecutive rows a warp examines at once (1..32)
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

// ---------------------------------------------------------------------------
// Production sampler: the sampled SET without the swap chain.
//
// For a slice of n entries with b = floor(c*n) draws r_j (j < b), let
//   T[t] = 1 + max{ j : r_j = t, j != t }   (0 when no such j).
// Because r_j >= j, a position t is only ever written by steps j <= t, so
// T[t] - 1 is the last step that moved a value INTO position t before step t
// and f(t) = T[t] ? f(T[t]-1) : t is the value sitting at position t when
// step t runs (chains strictly decrease).  The final content of positions
// [b, n) is the unpicked set, which gives
//   value t >= b is picked  <=>  T[t] != 0          (it was swapped out)
//   value v <  b is picked  <=>  v is not f(T[t]-1) for a targeted t >= b.
// Phase 1 only STORES T (highest lane wins within a chunk, program order
// across chunks), so there is no read-modify-write chain between chunks.
// Phase 2 marks the unpicked roots with a flag bit in T and emits the mask.
// Verified against the partial Fisher-Yates on 3000 random slices and by
// tests/test_gpu_parity.py::test_production_mask_equals_pick_sets.
// A chunk whose Lemire product might need the rejection loop switches the
// slice to an exact serial replay of the draws on lane 0.
// ---------------------------------------------------------------------------
// u16 / u32 max-store with the rare intra-instruction duplicate fixed up by CAS
__device__ __forceinline__ void tmax(uint16_t* T, uint32_t r, uint32_t v) {
  uint32_t* w = reinterpret_cast<uint32_t*>(reinterpret_cast<uintptr_t>(T + r) & ~uintptr_t(3));
  const uint32_t sh = (reinterpret_cast<uintptr_t>(T + r) & 2u) ? 16u : 0u;
  uint32_t old = *w;
  while (((old >> sh) & 0xffffu) < v) {
    const uint32_t nw = (old & ~(0xffffu << sh)) | (v << sh);
    const uint32_t got = atomicCAS(w, old, nw);
    if (got == old) break;
    old = got;
  }
}
__device__ __forceinline__ void tmax(uint32_t* T, uint32_t r, uint32_t v) { atomicMax(T + r, v); }


// Tiny slices (2 <= n <= kTinyCap): ONE LANE per slice runs the reference's
// partial Fisher-Yates itself (nmc.cpp:44-63 with the exact next_below of
// rng.hpp:32-45), its permutation in a 32-byte column of shared memory, and
// ORs the picked set into the mask.  The Zipf tails of configs 3 and 5 are
// millions of such slices (69 % of config 5's mode-0 rows): a warp per slice
// spends a chain of phase latencies on a handful of draws.
#ifndef NTCB_TINY_CAP
#define NTCB_TINY_CAP 64
#endif
constexpr uint32_t kTinyCap = NTCB_TINY_CAP;  // 32 or 64
constexpr uint64_t kTinyMin = 4096;  // tiny slices in a plan before the lane kernel is worth a launch
__global__ void __launch_bounds__(256) k_sample_tiny(SampleArgs a) {
  __shared__ unsigned char perm_s[kTinyCap * 256];  // [position][thread]
  unsigned char* pm = perm_s + threadIdx.x;
  for (uint64_t p = a.row_begin + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < a.row_end;
       p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t beg = a.off[p];
    const uint64_t n64 = a.off[p + 1] - beg;
    if (n64 < 2 || n64 > kTinyCap) continue;
    const uint32_t n = static_cast<uint32_t>(n64);
    const uint32_t b = static_cast<uint32_t>(blocksize_for(a.c, n));
    if (b == 0) continue;
    for (uint32_t i = 0; i < n; ++i) pm[i * 256] = static_cast<unsigned char>(i);
    uint64_t s = fork64(a.root, p);
    uint64_t set = 0;
    for (uint32_t j = 0; j < b; ++j) {
      const uint64_t bd = n - j;
      s += kGolden;
      uint64_t x = mix64(s);
      uint64_t lo = x * bd, hi = __umul64hi(x, bd);
      if (lo < bd) {  // rng.hpp:36-43
        const uint64_t th = (0 - bd) % bd;
        while (lo < th) {
          s += kGolden;
          x = mix64(s);
          lo = x * bd;
          hi = __umul64hi(x, bd);
        }
      }
      const uint32_t r = j + static_cast<uint32_t>(hi);
      const unsigned char pj = pm[j * 256], pr = pm[r * 256];
      pm[j * 256] = pr;
      pm[r * 256] = pj;
      set |= 1ull << pr;  // the pick: perm[j] after the swap
    }
    // the set's bits at absolute entry positions beg .. beg + n - 1 (up to three mask words)
    const uint32_t sh = static_cast<uint32_t>(beg & 31u);
    const uint32_t w0 = static_cast<uint32_t>(set << sh);
    const uint64_t rest = sh ? set >> (32u - sh) : set >> 32;  // bits from word 1 on
    uint32_t* m = a.mask + (beg >> 5);
    if (w0) atomicOr(m, w0);
    if (sh) {
      if (static_cast<uint32_t>(rest)) atomicOr(m + 1, static_cast<uint32_t>(rest));
      if (rest >> 32) atomicOr(m + 2, static_cast<uint32_t>(rest >> 32));
    } else if (static_cast<uint32_t>(rest)) {
      atomicOr(m + 1, static_cast<uint32_t>(rest));
    }
  }
}

template <typename TT>
__global__ void __launch_bounds__(kSampleWarps * 32) k_sample_set(SampleArgs a) {
  constexpr uint32_t FLAG = 1u << (8 * sizeof(TT) - 1);
  constexpr uint32_t VAL = FLAG - 1;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  TT* T = reinterpret_cast<TT*>(smem + static_cast<size_t>(wib) * a.warp_bytes);
  if (*reinterpret_cast<volatile unsigned long long*>(&a.counters[1]) != ~0ull) return;
  const uint64_t lane_off = static_cast<uint64_t>(lane + 1) * kGolden;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kSampleWarps;
  // The warp examines scan_w consecutive rows at once (one coalesced read of
  // their offsets) and then samples the ones of its class one by one: with a
  // Zipf tail most rows belong to k_sample_tiny, and skipping them one
  // dependent offset load at a time was most of this kernel's time.
  const uint32_t sw = a.scan_w;
  for (uint64_t base = a.row_begin + (blockIdx.x * static_cast<uint64_t>(kSampleWarps) + wib) * sw; base < a.row_end;
       base += nw * sw) {
   const uint64_t pl = base + lane;
   uint64_t beg_l = 0;
   uint32_t n_l = 0;
   if (static_cast<uint32_t>(lane) < sw && pl < a.row_end) {
     beg_l = a.off[pl];
     n_l = static_cast<uint32_t>(a.off[pl + 1] - beg_l);
   }
   const uint32_t b_l = static_cast<uint32_t>(blocksize_for(a.c, n_l));
   // skipped / full / heavy / tiny slices are not this kernel's
   uint32_t todo = __ballot_sync(kFull, !(b_l == 0 || a.c >= 1.0 || n_l > a.cap || n_l <= a.tiny_cap));
   while (todo) {
    const int tq = __ffs(todo) - 1;
    todo &= todo - 1;
    const uint64_t p = base + tq;
    const uint64_t beg = __shfl_sync(kFull, beg_l, tq);
    const uint32_t n = __shfl_sync(kFull, n_l, tq);
    const uint32_t b = __shfl_sync(kFull, b_l, tq);
    const uint64_t state0 = a.direct ? a.root : fork64(a.root, p);
    {
      const uint32_t pw = (n * static_cast<uint32_t>(sizeof(TT)) + 15) / 16;
      uint4* t4 = reinterpret_cast<uint4*>(T);
      for (uint32_t w = lane; w < pw; w += 32) t4[w] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();
    // ---- phase 1: draws (64 per step), last-writer stores ---------------------
    bool exact = false;
    uint64_t state = state0;
    for (uint32_t j0 = 0; j0 < b; j0 += 64) {
      uint32_t r[2], jj[2];
      bool act[2], ok = true;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        jj[h] = j0 + 32 * h + lane;
        act[h] = jj[h] < b;
        const uint32_t bound = act[h] ? n - jj[h] : 1u;
        const uint64_t x = mix64(state + lane_off + static_cast<uint64_t>(32 * h) * kGolden);
        const uint64_t t = static_cast<uint64_t>(static_cast<uint32_t>(x)) * bound;
        const uint64_t u = static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * bound + (t >> 32);
        ok = ok && !(act[h] && static_cast<uint32_t>(u) == 0u && static_cast<uint32_t>(t) < bound);
        r[h] = jj[h] + static_cast<uint32_t>(u >> 32);
      }
      if (__any_sync(kFull, !ok)) {
        exact = true;
        break;
      }
      state += 64 * kGolden;
      if (act[0] && r[0] != jj[0]) T[r[0]] = static_cast<TT>(jj[0] + 1);
      __syncwarp();
      if (act[1] && r[1] != jj[1]) T[r[1]] = static_cast<TT>(jj[1] + 1);
      __syncwarp();
      // two lanes of one store instruction with the same target: keep the max
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (act[h] && r[h] != jj[h] && static_cast<uint32_t>(T[r[h]]) < jj[h] + 1) tmax(T, r[h], jj[h] + 1);
      __syncwarp();
    }
    if (exact) {  // rare: replay every draw exactly (rng.hpp:32-45) on lane 0
      __syncwarp();
      const uint32_t pw = (n * static_cast<uint32_t>(sizeof(TT)) + 15) / 16;
      uint4* t4 = reinterpret_cast<uint4*>(T);
      for (uint32_t w = lane; w < pw; w += 32) t4[w] = make_uint4(0, 0, 0, 0);
      __syncwarp();
      if (lane == 0) {
        uint64_t s = state0;
        for (uint32_t j = 0; j < b; ++j) {
          const uint64_t bd = n - j;
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
          const uint32_t r = j + static_cast<uint32_t>(h2);
          if (r != j) T[r] = static_cast<TT>(j + 1);
        }
      }
      __syncwarp();
    }
    // ---- phase 2a: positions t in [b, n): bit t; mark unpicked roots -------
    // word k of the slice covers relative positions [32k - off0, 32k - off0 + 32)
    uint32_t* gm = a.mask + (beg >> 5);
    const int off0 = static_cast<int>(beg & 31u);
    const int kb0 = (static_cast<int>(b) + off0) >> 5;
    const int kend = (static_cast<int>(n) + off0 - 1) >> 5;
    if (b < n) {
      for (int k = kb0; k <= kend; ++k) {
        const int t = 32 * k - off0 + lane;
        const bool valid = t >= static_cast<int>(b) && t < static_cast<int>(n);
        const uint32_t tv = valid ? (static_cast<uint32_t>(T[t]) & VAL) : 0u;
        if (tv) {
          uint32_t v = tv - 1, nx;
          while ((nx = static_cast<uint32_t>(T[v]) & VAL) != 0u) v = nx - 1;
          T[v] = static_cast<TT>(FLAG);  // roots hold 0: the flag alone
        }
        const uint32_t bits = __ballot_sync(kFull, tv != 0u);
        if (lane == 0) {
          const bool whole = 32 * k - off0 >= static_cast<int>(b) && 32 * k - off0 + 32 <= static_cast<int>(n);
          if (whole)
            gm[k] = bits;
          else if (bits)
            atomicOr(&gm[k], bits);
        }
      }
    }
    __syncwarp();
    // ---- phase 2b: values v in [0, b): picked unless flagged ---------------
    const int kbend = (static_cast<int>(b) + off0 - 1) >> 5;
    for (int k = 0; k <= kbend; ++k) {
      const int t = 32 * k - off0 + lane;
      const bool pick = t >= 0 && t < static_cast<int>(b) && !(static_cast<uint32_t>(T[t]) & FLAG);
      const uint32_t bits = __ballot_sync(kFull, pick);
      if (lane == 0) {
        const bool whole = 32 * k - off0 >= 0 && 32 * k - off0 + 32 <= static_cast<int>(b);
        if (whole)
          gm[k] = bits;
        else if (bits)
          atomicOr(&gm[k], bits);
      }
    }
    __syncwarp();
   }
  }
}

// ---------------------------------------------------------------------------
// Mid-length slices (kWarpCap < n <= cap): the same set formulation with a
// whole CTA per slice, so a 10^4-entry slice is not one warp's serial
// chain-walk.  T is u32 in shared memory (4n bytes); phase 1 is one shared
// atomicMax per draw (order-free: the max is the last writer); the phases
// are separated by __syncthreads.  Slices are taken from a host-built list
// (longest first) through a device cursor, so CTAs stay busy to the end.
// ---------------------------------------------------------------------------

// 32-bit shared-window accesses: keeps the table base in one register
// instead of re-deriving the window from the CTA id at every access
__device__ __forceinline__ uint32_t ld_s(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_s(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
constexpr uint32_t kWarpCap = 1024;  // slices up to this length: warp per slice

struct CtaArgs {
  const uint64_t* off;
  const uint32_t* rows;  // slice list (view rows), longest first
  uint32_t n_rows;
  double c;
  uint64_t root;
  uint32_t* mask;
  unsigned long long* counters;  // [1] error key
  unsigned long long* cursor;    // zeroed before the launch
};

template <int kCtaThreads>
__global__ void __launch_bounds__(kCtaThreads) k_sample_cta(CtaArgs a) {
  constexpr uint32_t FLAG = 0x80000000u, VAL = 0x7fffffffu;
  constexpr int NW = kCtaThreads / 32;
  extern __shared__ __align__(16) uint32_t T[];
  __shared__ unsigned long long s_item;
  __shared__ int s_rej;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (*reinterpret_cast<volatile unsigned long long*>(&a.counters[1]) != ~0ull) return;
  while (true) {
    if (tid == 0) {
      s_item = atomicAdd(a.cursor, 1ull);
      s_rej = 0;
    }
    __syncthreads();
    const unsigned long long item = s_item;
    if (item >= a.n_rows) break;
    const uint64_t p = a.rows[item];
    const uint64_t beg = a.off[p];
    const uint32_t n = static_cast<uint32_t>(a.off[p + 1] - beg);
    const uint32_t b = static_cast<uint32_t>(blocksize_for(a.c, n));
    const uint64_t state0 = fork64(a.root, p);
    const uint32_t pw = (n + 3) / 4;
    uint4* t4 = reinterpret_cast<uint4*>(T);
    for (uint32_t w = tid; w < pw; w += kCtaThreads) t4[w] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    // ---- phase 1: T[r_j] = max(j + 1) over draws j with r_j != j ------------
    // (r_j == j stores max(T, 0): a no-op, so the atomic is unconditional).
    // A draw can need Lemire's rejection loop only if lo64(x * bound) < bound,
    // which requires the low word of u to be 0: track the minimum of those
    // words and replay the slice exactly if it ever hits 0 (p ~ b / 2^32).
    {
      uint32_t minu = 0xffffffffu;
      uint64_t s = state0 + static_cast<uint64_t>(tid + 1) * kGolden;
      auto draw = [&](uint32_t j, uint64_t st) {
        const uint32_t bound = n - j;
        const uint64_t x = mix64(st);
        const uint64_t t = static_cast<uint64_t>(static_cast<uint32_t>(x)) * bound;
        const uint64_t u = static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * bound + (t >> 32);
        minu = min(minu, static_cast<uint32_t>(u));
        const uint32_t r = j + static_cast<uint32_t>(u >> 32);
        atomicMax(&T[r], r != j ? j + 1 : 0u);
      };
      uint32_t j = tid;
      for (; j + kCtaThreads < b; j += 2 * kCtaThreads, s += 2 * kCtaThreads * kGolden) {
        draw(j, s);
        draw(j + kCtaThreads, s + kCtaThreads * kGolden);
      }
      if (j < b) draw(j, s);
      if (minu == 0u) s_rej = 1;
    }
    __syncthreads();
    if (s_rej) {  // rare: a draw may need Lemire's rejection loop -- exact serial replay
      for (uint32_t w = tid; w < pw; w += kCtaThreads) t4[w] = make_uint4(0, 0, 0, 0);
      __syncthreads();
      if (tid == 0) {
        uint64_t s = state0;
        for (uint32_t j = 0; j < b; ++j) {
          const uint64_t bd = n - j;
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
          const uint32_t r = j + static_cast<uint32_t>(h2);
          if (r != j) T[r] = j + 1;
        }
      }
      __syncthreads();
    }
    // ---- phase 2: a shared bitmap of the slice (word k covers relative
    // positions [32k - off0, 32k - off0 + 32)), pre-set to the values [0, b).
    // Positions t in [b, n) set their bit iff targeted (T[t] != 0) and clear
    // the bit of the unpicked root of their chain (a value < b); the two
    // kinds of bit never share a position, so OR and AND commute.  Then one
    // coalesced flush; only the slice's first and last words are shared with
    // neighbouring slices (atomicOr).
    const int off0 = static_cast<int>(beg & 31u);
    const int nw = (off0 + static_cast<int>(n) + 31) >> 5;
    uint32_t* SB = T + ((n + 3) & ~3u);  // after the table
    for (int k = tid; k < nw; k += kCtaThreads) {
      const int p0 = 32 * k - off0;  // relative position of bit 0
      const int lo_ = p0 < 0 ? -p0 : 0;                                   // first bit inside the slice
      const int hiv = static_cast<int>(b) - p0;                           // bits below b
      const uint32_t below = hiv <= 0 ? 0u : hiv >= 32 ? 0xffffffffu : ((1u << hiv) - 1u);
      SB[k] = below & (0xffffffffu << lo_);
    }
    __syncthreads();
    {
      uint32_t tb;  // opaque copy: ptxas would otherwise re-derive it per access
      asm volatile("mov.u32 %0, %1;" : "=r"(tb) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(T))));
      const int kb0 = (static_cast<int>(b) + off0) >> 5;
      const int kend = nw - 1;
      const uint32_t span = n - b;
      for (int k = kb0 + wid; k <= kend; k += NW) {
        const int t = 32 * k - off0 + lane;
        const uint32_t tv = static_cast<uint32_t>(t - static_cast<int>(b)) < span ? (ld_s(tb + 4u * t) & VAL) : 0u;
        if (tv) {
          uint32_t a4 = tb + 4u * (tv - 1), nx;
          while ((nx = ld_s(a4) & VAL) != 0u) a4 = tb + 4u * (nx - 1);
          const uint32_t v = (a4 - tb) >> 2;  // the unpicked root (< b)
          atomicAnd(&SB[(static_cast<uint32_t>(off0) + v) >> 5], ~(1u << ((static_cast<uint32_t>(off0) + v) & 31u)));
        }
        const uint32_t bits = __ballot_sync(kFull, tv != 0u);
        if (lane == 0 && bits) atomicOr(&SB[k], bits);
      }
    }
    __syncthreads();
    uint32_t* gm = a.mask + (beg >> 5);
    for (int k = tid; k < nw; k += kCtaThreads) {
      const uint32_t v = SB[k];
      if (k != 0 && k != nw - 1)
        gm[k] = v;
      else if (v)
        atomicOr(&gm[k], v);
    }
    __syncthreads();
  }
}

// Per (view, row range, cap): how many short slices, and the mid-slice lists
// in two size buckets (small tables -> many CTAs per SM; large tables -> 1024
// threads per slice), longest first.
constexpr uint32_t kMidSplit = 16384;
struct SampleBucket {
  uint32_t* rows = nullptr;
  uint32_t n = 0;
  uint32_t max_len = 0;
};
struct SamplePlan {
  uint64_t n_short = 0;
  uint64_t n_tiny = 0;  // of those, slices of at most kTinyCap entries
  SampleBucket mid[2];
};
using SamplePlans = std::map<std::tuple<const void*, uint64_t, uint64_t, uint64_t>, SamplePlan>;

static const SamplePlan& sample_plan(ntcb_context* ctx, const DeviceView& v, uint64_t r0, uint64_t r1,
                                     uint64_t cap) {
  auto& g_splans = ctx_cache<SamplePlans>(ctx, kCacheSample);
  auto key = std::make_tuple(static_cast<const void*>(v.off), r0, r1, cap);
  auto it = g_splans.find(key);
  if (it != g_splans.end()) return it->second;
  SamplePlan pl;
  std::vector<std::pair<uint64_t, uint32_t>> mid[2];
  for (uint64_t p = r0; p < r1; ++p) {
    const uint64_t n = v.h_off[p + 1] - v.h_off[p];
    if (n < 2) continue;  // b = floor(c n) = 0 for c < 1
    if (n <= kTinyCap) ++pl.n_tiny;
    if (n <= kWarpCap)
      ++pl.n_short;
    else if (n <= cap)
      mid[n > kMidSplit].emplace_back(n, static_cast<uint32_t>(p));
  }
  for (int k = 0; k < 2; ++k) {
    auto& m = mid[k];
    std::stable_sort(m.begin(), m.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    if (m.empty()) continue;
    std::vector<uint32_t> rows(m.size());
    for (size_t i = 0; i < m.size(); ++i) rows[i] = m[i].second;
    NTCB_CUDA(cudaMalloc(&pl.mid[k].rows, sizeof(uint32_t) * rows.size()));
    NTCB_CUDA(cudaMemcpy(pl.mid[k].rows, rows.data(), sizeof(uint32_t) * rows.size(), cudaMemcpyHostToDevice));
    pl.mid[k].n = static_cast<uint32_t>(rows.size());
    pl.mid[k].max_len = static_cast<uint32_t>(m.front().first);
  }
  return g_splans.emplace(key, pl).first->second;
}

template <int T>
static void launch_cta_bucket(ntcb_context* ctx, cudaStream_t stream, const SampleBucket& bk, CtaArgs a) {
  a.rows = bk.rows;
  a.n_rows = bk.n;
  // u32 table (padded to 16 bytes) + the slice bitmap (off0 + n bits)
  const size_t smem = (static_cast<size_t>(bk.max_len) + 3) / 4 * 16 + ((bk.max_len + 31) / 32 + 2) * 4;
  NTCB_CUDA(cudaFuncSetAttribute(k_sample_cta<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  int per_sm = 0;
  NTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sample_cta<T>, T, smem));
  if (per_sm < 1) per_sm = 1;
  const int side_cap = ctx->tune.side_sampler_ctas;  // tuning knob (ntcb_tuning)
  if (stream == ctx->side && side_cap > 0) per_sm = std::min(per_sm, side_cap);
  const uint64_t grid = std::min<uint64_t>(bk.n, static_cast<uint64_t>(per_sm) * ctx->sm_count);
  NTCB_CUDA(cudaMemsetAsync(a.cursor, 0, sizeof(unsigned long long), stream));
  k_sample_cta<T><<<static_cast<unsigned>(grid), T, smem, stream>>>(a);
  NTCB_CUDA(cudaGetLastError());
}

// Short slices on the warp kernel, mid slices on the CTA kernel; returns the
// number of launches and the cap above which launch_sample_heavy takes over.
int launch_sample_set(ntcb_context* ctx, cudaStream_t stream, uint32_t* mask, int mode,
                      uint64_t row_begin, uint64_t row_end, double c, uint64_t root, int direct,
                      uint64_t* heavy_cap) {
  const DeviceView& v = ctx->views[mode];
  if (heavy_cap) *heavy_cap = ~0ull;
  if (row_end <= row_begin || c >= 1.0) return 0;
  if (v.max_slice >= (1ull << 31))
    fail(NTCB_EINVAL, "sampler: slices of 2^31 or more entries are not supported");
  // shared-memory cap of the CTA kernel: u32 per entry, <= 48K entries
  uint64_t cap = std::min<uint64_t>(v.max_slice, 49152);
  if (cap < kWarpCap) cap = kWarpCap;
  if (heavy_cap) *heavy_cap = cap;
  const SamplePlan& pl = sample_plan(ctx, v, row_begin, row_end, cap);
  int launches = 0;
  if (pl.n_short) {
    SampleArgs a{};
    a.off = v.off;
    a.row_begin = row_begin;
    a.row_end = row_end;
    a.c = c;
    a.root = root;
    a.mask = mask;
    a.counters = ctx->counters;
    a.direct = direct;
    a.cap = std::min<uint64_t>(v.max_slice, kWarpCap);
    // the Zipf tail: a lane per slice instead of a warp per slice
    const bool tiny = !direct && ctx->tune.tiny_sampler != 0 && pl.n_tiny >= kTinyMin;
    a.tiny_cap = tiny ? kTinyCap : 0u;
    if (tiny) {
      const uint64_t rows = row_end - row_begin;
      const uint64_t tg = std::min<uint64_t>((rows + 255) / 256, static_cast<uint64_t>(ctx->sm_count) * 8);
      k_sample_tiny<<<static_cast<unsigned>(tg), 256, 0, stream>>>(a);
      NTCB_CUDA(cudaGetLastError());
      ++launches;
    }
    a.warp_bytes = static_cast<uint32_t>((a.cap * 2 + 15) / 16 * 16);
    const size_t smem = static_cast<size_t>(a.warp_bytes) * kSampleWarps;
    int per_sm = 0;
    NTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sample_set<uint16_t>,
                                                            kSampleWarps * 32, smem));
    if (per_sm < 1) per_sm = 1;
    // rows examined per warp step: as wide as leaves every resident warp at least four steps
    const uint64_t resident = static_cast<uint64_t>(per_sm) * ctx->sm_count * kSampleWarps;
    a.scan_w = 1;
    while (a.scan_w < 32 && (row_end - row_begin) / (2ull * a.scan_w) >= 4 * resident) a.scan_w *= 2;
    uint64_t grid = ((row_end - row_begin + a.scan_w - 1) / a.scan_w + kSampleWarps - 1) / kSampleWarps;
    grid = std::min<uint64_t>(grid, static_cast<uint64_t>(per_sm) * ctx->sm_count);
    k_sample_set<uint16_t><<<static_cast<unsigned>(grid), kSampleWarps * 32, smem, stream>>>(a);
    NTCB_CUDA(cudaGetLastError());
    ++launches;
  }
  for (int k = 0; k < 2; ++k) {
    if (!pl.mid[k].n) continue;
    if (direct) fail(NTCB_EINVAL, "sampler: direct streams are single-slice (warp kernel)");
    CtaArgs a{};
    a.off = v.off;
    a.c = c;
    a.root = root;
    a.mask = mask;
    a.counters = ctx->counters;
    // one cursor per (stream, bucket): the buckets run back to back on one stream
    a.cursor = ctx->counters + (stream == ctx->side ? 4 : 6) + k;
    if (k == 0)
      launch_cta_bucket<256>(ctx, stream, pl.mid[k], a);
    else
      launch_cta_bucket<1024>(ctx, stream, pl.mid[k], a);
    ++launches;
  }
  return launches;
}

void drop_sample_plans(ntcb_context* ctx) {
  if (!ctx->cache[kCacheSample]) return;
  for (auto& kv : ctx_cache<SamplePlans>(ctx, kCacheSample))
    for (auto& b : kv.second.mid)
      if (b.rows) cudaFree(b.rows);
  ctx_cache_free<SamplePlans>(ctx, kCacheSample);
}

// ---------------------------------------------------------------------------
// Heavy slices (n above the per-warp shared-memory budget): the same set
// formulation over the whole grid.  T lives in the per-entry u32 scratch
// (T[t] of slice p at scratch[beg + t], flag bit 31); kernel boundaries are
// the phase barriers; last-writer becomes atomicMax.  Slices where a draw
// might need Lemire's rejection loop are flagged and redone by the exact
// ordered warp sampler (fy_slice on the global scratch).
// ---------------------------------------------------------------------------
struct HeavyRow {
  uint64_t row, beg;
  uint32_t n, b;
  uint64_t tb;  // word offset of the slice's bitmaps in the plan's bit buffer: tb[ceil(b/32)], then rb
};

__global__ void k_heavy_zero(const HeavyRow* rows, uint32_t* scratch, int* flags) {
  const HeavyRow h = rows[blockIdx.y];
  if (blockIdx.x == 0 && threadIdx.x == 0) flags[blockIdx.y] = 0;
  // 16-byte stores over the aligned body, 4-byte ones at the two ends
  uint32_t* p = scratch + h.beg;
  const uint32_t mis = static_cast<uint32_t>((4 - (h.beg & 3)) & 3);
  const uint32_t head = mis < h.n ? mis : h.n;
  const uint32_t body4 = (h.n - head) >> 2;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  if (tid < head) p[tid] = 0u;
  uint4* q = reinterpret_cast<uint4*>(p + head);
  for (uint32_t t = tid; t < body4; t += nth) q[t] = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t tail0 = head + 4 * body4;
  if (tid < h.n - tail0) p[tail0 + tid] = 0u;
}

// Head phase, one mask word per lane: picked = not an unpicked root, i.e.
// the complement of the slice's rb bits (b bits; bit v = head position v)
// aligned to the word's absolute entry positions.
__device__ __forceinline__ void head_words(const HeavyRow& h, const uint32_t* rb, uint32_t* mask, uint64_t tid,
                                           uint64_t nth) {
  const uint64_t ga0 = h.beg, ga1 = h.beg + h.b;
  const uint64_t w0 = ga0 >> 5, w1 = (ga1 - 1) >> 5;
  for (uint64_t w = w0 + tid; w <= w1; w += nth) {
    const int64_t o = static_cast<int64_t>(w << 5) - static_cast<int64_t>(h.beg);  // rb bit of the word's entry 0
    uint32_t win;
    if (o >= 0) {
      const uint64_t k = static_cast<uint64_t>(o) >> 5;
      const uint32_t s = static_cast<uint32_t>(o) & 31u;
      win = s ? (rb[k] >> s) | (rb[k + 1] << (32 - s)) : rb[k];
    } else {
      win = rb[0] << static_cast<uint32_t>(-o);
    }
    uint32_t valid = ~0u;
    if ((w << 5) < ga0) valid &= ~0u << (ga0 - (w << 5));
    if ((w << 5) + 32 > ga1) valid &= ~0u >> ((w << 5) + 32 - ga1);
    const uint32_t picked = ~win & valid;
    if (valid == ~0u)
      mask[w] = picked;
    else if (picked)
      atomicOr(&mask[w], picked);
  }
}

// Draw phase.  Besides T, a head position r < b that a draw targets gets its
// bit in the slice's L2-resident bitmap tb (T[r] != 0), which the tail
// phase consults before touching the table.
__global__ void k_heavy_draw(const HeavyRow* rows, uint32_t* scratch, int* flags, uint64_t root,
                             int direct) {
  const HeavyRow h = rows[blockIdx.y];
  const uint64_t state = direct ? root : fork64(root, h.row);
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < h.b; j += gridDim.x * blockDim.x) {
    const uint32_t bound = h.n - j;
    const uint64_t x = mix64(state + static_cast<uint64_t>(j + 1) * kGolden);
    const uint64_t t = static_cast<uint64_t>(static_cast<uint32_t>(x)) * bound;
    const uint64_t u = static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * bound + (t >> 32);
    if (static_cast<uint32_t>(u) == 0u && static_cast<uint32_t>(t) < bound) flags[blockIdx.y] = 1;
    const uint32_t r = j + static_cast<uint32_t>(u >> 32);
    if (r != j) atomicMax(&scratch[h.beg + r], j + 1);
  }
}

// tb (T[v] != 0 for head positions v < b) of every heavy slice, from the
// finished table in one streaming pass (a warp per 32 positions) -- cheaper
// than an L2 atomicOr per head-targeting draw.
__global__ void k_heavy_tb(const HeavyRow* rows, const uint32_t* scratch, const int* flags, uint32_t* bits) {
  const HeavyRow h = rows[blockIdx.y];
  if (flags[blockIdx.y] || h.b == 0) return;
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (static_cast<uint64_t>(h.b) + 31) / 32;
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  uint32_t* tb = bits + h.tb;
  constexpr int kIlp = 8;  // words per warp step: 8 loads in flight per lane
  for (uint64_t w0 = blockIdx.x * static_cast<uint64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); w0 < nw;
       w0 += kIlp * nwarps) {
    uint32_t t[kIlp];
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
      const uint64_t v = ((w0 + i * nwarps) << 5) + lane;
      t[i] = v < h.b ? scratch[h.beg + v] : 0u;
    }
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
      const uint32_t word = __ballot_sync(kFull, (t[i] & 0x7fffffffu) != 0u);
      if (lane == 0 && w0 + i * nwarps < nw) tb[w0 + i * nwarps] = word;
    }
  }
}

// Chain walks are dependent reads: each warp takes kTailIlp mask words at
// once and walks their chains in lockstep (kTailIlp independent reads in
// flight per lane).  Chains are disjoint (the last draw targeting a position
// is unique to it), so each root has one writer.
constexpr int kTailIlp = 4;

// Giant slices, bucketed draw phase: the draws are sorted by target window
// (kernel boundaries between the passes), so every draw is computed twice --
// once to count, once to scatter -- instead of once per window it could
// reach (r_j >= j: window k needs every j < w1, 12x the draws for a
// 261M-entry slice), and each window's bucket is then applied with
// L2-resident atomics.  Pass 1: per-CTA histograms over a fixed j range.
constexpr int kGiantCtas = 1184;  // 8 x 148: CTAs of the count / scatter passes
__device__ __forceinline__ uint32_t giant_draw(uint64_t state, uint32_t j, uint32_t n, bool& rej) {
  const uint32_t bound = n - j;
  const uint64_t x = mix64(state + static_cast<uint64_t>(j + 1) * kGolden);
  const uint64_t t = static_cast<uint64_t>(static_cast<uint32_t>(x)) * bound;
  const uint64_t u = static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * bound + (t >> 32);
  rej = static_cast<uint32_t>(u) == 0u && static_cast<uint32_t>(t) < bound;
  return j + static_cast<uint32_t>(u >> 32);
}
__global__ void __launch_bounds__(256) k_giant_count(const HeavyRow* rows, int* flags, uint64_t root, int direct,
                                                     int wlog, int nwin, uint32_t* hist /*[nwin][ctas]*/) {
  __shared__ uint32_t sh[256];
  const HeavyRow h = rows[0];
  const uint64_t state = direct ? root : fork64(root, h.row);
  for (int i = threadIdx.x; i < nwin; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t per = (h.b + gridDim.x - 1) / gridDim.x;
  const uint32_t j0 = blockIdx.x * per, j1 = min(h.b, j0 + per);
  bool any_rej = false;
  for (uint32_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    bool rej;
    const uint32_t r = giant_draw(state, j, h.n, rej);
    any_rej |= rej;
    if (r != j) atomicAdd(&sh[r >> wlog], 1u);
  }
  if (any_rej) flags[0] = 1;
  __syncthreads();
  for (int i = threadIdx.x; i < nwin; i += blockDim.x) hist[static_cast<uint64_t>(i) * gridDim.x + blockIdx.x] = sh[i];
}
// Pass 2: exclusive scan of hist in (window, CTA) order (one CTA) -> scatter
// offsets; wbeg[w] = the first pair of window w (wbeg[nwin] = total).
__global__ void __launch_bounds__(1024) k_giant_scan(uint32_t* hist, uint32_t n, int nwin, int ctas, uint32_t* wbeg) {
  __shared__ uint32_t part[1024];
  const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint32_t a = threadIdx.x * per, b = min(n, a + per);
  uint32_t s = 0;
  for (uint32_t i = a; i < b; ++i) s += hist[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (uint32_t t = 0; t < blockDim.x; ++t) {
      const uint32_t v = part[t];
      part[t] = run;
      run += v;
    }
  }
  __syncthreads();
  uint32_t run = part[threadIdx.x];
  for (uint32_t i = a; i < b; ++i) {
    const uint32_t v = hist[i];
    hist[i] = run;
    if (i % ctas == 0) wbeg[i / ctas] = run;
    run += v;
  }
  if (threadIdx.x == blockDim.x - 1) wbeg[nwin] = run;
}
// Pass 3: the same draws again, scattered as (r, j + 1) into their window's bucket.
__global__ void __launch_bounds__(256) k_giant_scatter(const HeavyRow* rows, uint64_t root, int direct, int wlog,
                                                       int nwin, const uint32_t* hist, uint2* pairs) {
  __shared__ uint32_t cur[256];
  const HeavyRow h = rows[0];
  const uint64_t state = direct ? root : fork64(root, h.row);
  for (int i = threadIdx.x; i < nwin; i += blockDim.x) cur[i] = hist[static_cast<uint64_t>(i) * gridDim.x + blockIdx.x];
  __syncthreads();
  const uint32_t per = (h.b + gridDim.x - 1) / gridDim.x;
  const uint32_t j0 = blockIdx.x * per, j1 = min(h.b, j0 + per);
  for (uint32_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    bool rej;
    const uint32_t r = giant_draw(state, j, h.n, rej);
    if (r != j) pairs[atomicAdd(&cur[r >> wlog], 1u)] = make_uint2(r, j + 1);
  }
}
// Pass 4 (one launch per window): T[r] = max(T[r], j + 1) in L2, and the
// head-position bitmap tb (r < b: T[r] != 0).
__global__ void k_giant_apply(const HeavyRow* rows, const uint2* pairs, const uint32_t* wbeg, int w,
                              uint32_t* scratch) {
  const HeavyRow h = rows[0];
  const uint32_t p0 = wbeg[w], p1 = wbeg[w + 1];
  for (uint32_t i = p0 + blockIdx.x * blockDim.x + threadIdx.x; i < p1; i += gridDim.x * blockDim.x) {
    const uint2 q = pairs[i];
    atomicMax(&scratch[h.beg + q.x], q.y);
  }
}

// Tail and head phases of one slice longer than the draw window.  Chain
// steps consult the L2-resident bitmap `tb` (bit v: T[v] != 0, v < b) before
// touching the DRAM-resident table, so the ~3/4 of chains that end at their
// first node cost no random DRAM read; roots go to the bitmap `rb` (atomicOr
// in L2) instead of bit 31 of the table, and the head phase reads `rb`.
__global__ void k_heavy_tail_big(const HeavyRow* rows, const uint32_t* scratch, const int* flags, uint32_t* mask,
                                 const uint32_t* tb, uint32_t* rb) {
  const HeavyRow h = rows[0];
  if (flags[0]) return;
  const uint64_t gb0 = h.beg + h.b, gb1 = h.beg + h.n;
  if (gb1 <= gb0) return;
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = gb0 >> 5, w1 = (gb1 - 1) >> 5;
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  const uint32_t* sc = scratch + h.beg;
  for (uint64_t w = w0 + (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)); w <= w1; w += nwarps) {
    const uint64_t g = (w << 5) + lane;
    const bool valid = g >= gb0 && g < gb1;
    const uint32_t tv = valid ? (scratch[g] & 0x7fffffffu) : 0u;
    if (tv) {
      uint32_t v = tv - 1;
      while ((tb[v >> 5] >> (v & 31u)) & 1u) v = (sc[v] & 0x7fffffffu) - 1;
      atomicOr(&rb[v >> 5], 1u << (v & 31u));  // unpicked root (chains are disjoint)
    }
    const uint32_t bits = __ballot_sync(kFull, tv != 0u);
    if (lane == 0) {
      if ((w << 5) >= gb0 && (w << 5) + 32 <= gb1)
        mask[w] = bits;
      else if (bits)
        atomicOr(&mask[w], bits);
    }
  }
}

__global__ void k_heavy_head_big(const HeavyRow* rows, const int* flags, uint32_t* mask, const uint32_t* rb) {
  const HeavyRow h = rows[0];
  if (flags[0] || h.b == 0) return;
  head_words(h, rb, mask, blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x,
             static_cast<uint64_t>(gridDim.x) * blockDim.x);
}

__global__ void k_heavy_tail(const HeavyRow* rows, const uint32_t* scratch, const int* flags,
                             uint32_t* mask, uint32_t* bits) {
  const HeavyRow h = rows[blockIdx.y];
  if (flags[blockIdx.y]) return;
  const uint64_t gb0 = h.beg + h.b, gb1 = h.beg + h.n;
  if (gb1 <= gb0) return;
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = gb0 >> 5, w1 = (gb1 - 1) >> 5;
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  const uint32_t* sc = scratch + h.beg;
  const uint32_t* tb = bits + h.tb;
  uint32_t* rb = bits + h.tb + (static_cast<uint64_t>(h.b) + 31) / 32;
  for (uint64_t wb = w0 + (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)); wb <= w1;
       wb += kTailIlp * nwarps) {
    uint32_t v[kTailIlp];
    bool walk[kTailIlp];
#pragma unroll
    for (int i = 0; i < kTailIlp; ++i) {
      const uint64_t w = wb + i * nwarps;
      const uint64_t g = (w << 5) + lane;
      const bool valid = w <= w1 && g >= gb0 && g < gb1;
      const uint32_t tv = valid ? (scratch[g] & 0x7fffffffu) : 0u;
      walk[i] = tv != 0u;
      v[i] = tv - 1;
      const uint32_t bits32 = __ballot_sync(kFull, walk[i]);
      if (lane == 0 && w <= w1) {
        if ((w << 5) >= gb0 && (w << 5) + 32 <= gb1)
          mask[w] = bits32;
        else if (bits32)
          atomicOr(&mask[w], bits32);
      }
    }
    // chains: v -> T[v] - 1 while T[v] != 0 (tb bit set; ~3/4 of the chains
    // end at their first node and never read the DRAM-resident table); the
    // unpicked root goes to the bitmap rb (chains are disjoint: one writer)
    bool any = true;
    while (any) {
      bool cont[kTailIlp];
#pragma unroll
      for (int i = 0; i < kTailIlp; ++i) cont[i] = walk[i] && ((tb[v[i] >> 5] >> (v[i] & 31u)) & 1u);
      uint32_t nx[kTailIlp];
#pragma unroll
      for (int i = 0; i < kTailIlp; ++i) nx[i] = cont[i] ? (sc[v[i]] & 0x7fffffffu) : 0u;
      any = false;
#pragma unroll
      for (int i = 0; i < kTailIlp; ++i) {
        if (!walk[i]) continue;
        if (cont[i]) {
          v[i] = nx[i] - 1;
          any = true;
        } else {
          atomicOr(&rb[v[i] >> 5], 1u << (v[i] & 31u));
          walk[i] = false;
        }
      }
    }
  }
}

__global__ void k_heavy_head(const HeavyRow* rows, const int* flags, uint32_t* mask, const uint32_t* bits) {
  const HeavyRow h = rows[blockIdx.y];
  if (flags[blockIdx.y] || h.b == 0) return;
  head_words(h, bits + h.tb + (static_cast<uint64_t>(h.b) + 31) / 32, mask,
             blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x,
             static_cast<uint64_t>(gridDim.x) * blockDim.x);
}

// exact ordered fallback for flagged heavy slices (one warp each)
__global__ void k_heavy_exact(const HeavyRow* rows, uint32_t* scratch, const int* flags,
                              uint32_t* mask, uint64_t root, int direct) {
  __shared__ int tgt[32];
  __shared__ uint32_t rtmp[32];
  const HeavyRow h = rows[blockIdx.x];
  if (!flags[blockIdx.x]) return;
  const int lane = threadIdx.x & 31;
  uint32_t* gp = scratch + h.beg;
  for (uint32_t t = lane; t < h.n; t += 32) gp[t] = 0u;
  __syncwarp();
  fy_slice<uint32_t, false>(gp, h.n, h.b, direct ? root : fork64(root, h.row), lane, tgt, rtmp,
                            nullptr, mask, h.beg, nullptr);
}

constexpr uint32_t kMidSlice = 1u << 20;
struct HeavyPlan {
  HeavyRow* rows;   // device copy of the slice list (order below)
  uint32_t n;       // slices
  uint64_t maxn;    // longest slice
  uint32_t n_reg;   // slices [0, n_reg) draw in one pass; the rest (host copies in `giant`) by windows
  uint32_t n_small = 0;                  // [0, n_small): n <= kMidSlice; [n_small, n_reg): mid slices
  uint64_t max_small = 0, max_mid = 0;
  std::vector<HeavyRow> giant;
  uint32_t* bits = nullptr;       // per giant slice: tb and rb bitmaps over [0, b)
  std::vector<uint64_t> bit_off;  // word offset of giant slice i's tb (rb follows)
  uint64_t bit_words = 0;
  uint2* pairs = nullptr;     // bucketed draws of one giant slice (b_max pairs)
  uint32_t* ghist = nullptr;  // [windows][kGiantCtas] histograms / scatter offsets, then wbeg
};
// slice length above which the bitmap path runs / the draw window (entries),
// from the context's tuning (log2, validated to [16, 30] by ntcb_set_tuning)
static uint32_t heavy_big(const ntcb_context* ctx) { return 1u << ctx->tune.heavy_big_log2; }
static uint32_t heavy_window(const ntcb_context* ctx) { return 1u << ctx->tune.heavy_win_log2; }
using HeavyPlans = std::map<std::tuple<const void*, uint64_t, uint64_t, uint64_t, uint64_t>, HeavyPlan>;

int launch_sample_heavy(ntcb_context* ctx, cudaStream_t stream, uint32_t* mask, int mode,
                        uint64_t row_begin, uint64_t row_end, double c, uint64_t root, int direct,
                        uint64_t cap) {
  const DeviceView& v = ctx->views[mode];
  if (v.max_slice <= cap || c >= 1.0) return 0;
  uint64_t cbits;
  std::memcpy(&cbits, &c, 8);
  auto& g_heavy = ctx_cache<HeavyPlans>(ctx, kCacheHeavy);
  auto key = std::make_tuple(static_cast<const void*>(v.off), row_begin, row_end, cbits, cap);
  auto it = g_heavy.find(key);
  if (it == g_heavy.end()) {
    std::vector<HeavyRow> hr;
    uint32_t maxn = 0;
    for (uint64_t p = row_begin; p < row_end; ++p) {
      const uint64_t n = v.h_off[p + 1] - v.h_off[p];
      const uint64_t b = blocksize_for(c, n);
      if (n > cap && b > 0) {
        hr.push_back({p, v.h_off[p], static_cast<uint32_t>(n), static_cast<uint32_t>(b), 0});
        maxn = std::max<uint32_t>(maxn, static_cast<uint32_t>(n));
      }
    }
    // order: small slices, then mid slices (> kMidSlice: launched with wider
    // grids so fewer of their tables are in flight at once, L2 footprint),
    // then slices whose table is too long to stay in L2 alongside its
    // neighbours (windowed draws, bitmap-assisted tail and head, one per launch)
    const uint32_t big = std::min(heavy_big(ctx), heavy_window(ctx));
    std::stable_partition(hr.begin(), hr.end(), [](const HeavyRow& h) { return h.n <= kMidSlice; });
    std::stable_partition(hr.begin(), hr.end(), [big](const HeavyRow& h) { return h.n <= big; });
    HeavyPlan pl{nullptr, static_cast<uint32_t>(hr.size()), maxn, 0, {}};
    for (const HeavyRow& h : hr) {
      if (h.n <= big) {
        ++pl.n_reg;
        if (h.n <= kMidSlice) {
          ++pl.n_small;
          pl.max_small = std::max<uint64_t>(pl.max_small, h.n);
        } else {
          pl.max_mid = std::max<uint64_t>(pl.max_mid, h.n);
        }
      } else {
        pl.giant.push_back(h);
      }
    }
    // every slice: head bitmaps tb (T != 0) and rb (unpicked roots), b bits each
    for (HeavyRow& h : hr) {
      h.tb = pl.bit_words;
      pl.bit_words += 2 * ((static_cast<uint64_t>(h.b) + 31) / 32);
    }
    for (size_t i = 0; i < pl.giant.size(); ++i) {
      pl.giant[i].tb = hr[pl.n_reg + i].tb;
      pl.bit_off.push_back(pl.giant[i].tb);
    }
    if (pl.bit_words) NTCB_CUDA(cudaMalloc(&pl.bits, sizeof(uint32_t) * (pl.bit_words + 1)));  // +1: window reads
    if (!pl.giant.empty()) {
      uint64_t bmax = 0, nmax = 0;
      for (const HeavyRow& h : pl.giant) {
        bmax = std::max<uint64_t>(bmax, h.b);
        nmax = std::max<uint64_t>(nmax, h.n);
      }
      const uint64_t nwin = (nmax + heavy_window(ctx) - 1) / heavy_window(ctx);
      if (nwin > 256) fail(NTCB_EINVAL, "sampler: more than 256 draw windows in one slice");
      NTCB_CUDA(cudaMalloc(&pl.pairs, sizeof(uint2) * std::max<uint64_t>(bmax, 1)));
      NTCB_CUDA(cudaMalloc(&pl.ghist, sizeof(uint32_t) * (nwin * kGiantCtas + nwin + 1)));
    }
    if (!hr.empty()) {
      NTCB_CUDA(cudaMalloc(&pl.rows, sizeof(HeavyRow) * (hr.size() + 1)));
      NTCB_CUDA(cudaMemcpy(pl.rows, hr.data(), sizeof(HeavyRow) * hr.size(), cudaMemcpyHostToDevice));
    }
    it = g_heavy.emplace(key, std::move(pl)).first;
  }
  const uint32_t nh = it->second.n;
  if (nh == 0) return 0;
  if (nh > 65535) fail(NTCB_EINVAL, "sampler: more than 65535 heavy slices in one call");
  if (!view_scratch(ctx, mode)) fail(NTCB_ECUDA, "sampler: heavy slices need the per-entry scratch");
  if (ctx->heavy_flags_n < nh) {
    if (ctx->heavy_flags) cudaFree(ctx->heavy_flags);
    NTCB_CUDA(cudaMalloc(&ctx->heavy_flags, sizeof(int) * nh));
    ctx->heavy_flags_n = nh;
  }
  const HeavyRow* d = it->second.rows;
  // (chunk, slice) grids: 2 x SMs CTAs per slice at most, fewer when the
  // longest slice gives each thread less than ~kPer entries -- slices of a
  // few hundred thousand entries otherwise launch ~300 mostly idle CTAs
  // each (config 4: 1000 slices of 500K entries, CTA-launch bound; kPer = 8 measured
  // best: config 4 tail phase 5.06 -> 2.40 ms per mode).
  // ntcb_tuning.heavy_per overrides kPer for experiments.
  const uint64_t per = static_cast<uint64_t>(ctx->tune.heavy_per);
  const uint64_t maxn = it->second.maxn;
  auto gx = [&](uint64_t work) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(ctx->sm_count * 2, (work + 256 * per - 1) / (256 * per))));
  };
  const dim3 gz(gx((maxn + 3) / 4), nh);  // 16-byte stores
  k_heavy_zero<<<gz, 256, 0, stream>>>(d, view_scratch(ctx, mode), ctx->heavy_flags);
  if (it->second.bit_words)
    NTCB_CUDA(cudaMemsetAsync(it->second.bits, 0, sizeof(uint32_t) * it->second.bit_words, stream));
  const uint32_t n_reg = it->second.n_reg;
  int launches = 2;  // zero, exact
  const HeavyPlan& hp = it->second;
  // per size class: rows [r0, r0 + cnt), longest mx, grid cap
  struct Cls {
    uint32_t r0, cnt;
    uint64_t mx;
    uint64_t cap;
  };
  const Cls cls[2] = {{0, hp.n_small, hp.max_small, static_cast<uint64_t>(ctx->sm_count) * 2},
                      {hp.n_small, n_reg - hp.n_small, hp.max_mid, static_cast<uint64_t>(ctx->sm_count) * 8}};
  auto gxc = [&](const Cls& c, uint64_t work) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(c.cap, (work + 256 * per - 1) / (256 * per))));
  };
  for (const Cls& c : cls) {
    if (!c.cnt) continue;
    k_heavy_draw<<<dim3(gxc(c, (c.mx + 1) / 2), c.cnt), 256, 0, stream>>>(d + c.r0, view_scratch(ctx, mode),
                                                                          ctx->heavy_flags + c.r0, root, direct);
    ++launches;
  }
  for (size_t i = 0; i < hp.giant.size(); ++i) {
    const HeavyRow& h = hp.giant[i];
    const int wlog = ctx->tune.heavy_win_log2;
    const int nwin = static_cast<int>((static_cast<uint64_t>(h.n) + (1ull << wlog) - 1) >> wlog);
    const HeavyRow* dr = d + n_reg + i;
    uint32_t* wbeg = hp.ghist + static_cast<uint64_t>(nwin) * kGiantCtas;
    k_giant_count<<<kGiantCtas, 256, 0, stream>>>(dr, ctx->heavy_flags + n_reg + i, root, direct, wlog, nwin,
                                                  hp.ghist);
    k_giant_scan<<<1, 1024, 0, stream>>>(hp.ghist, static_cast<uint32_t>(nwin) * kGiantCtas, nwin, kGiantCtas,
                                         wbeg);
    k_giant_scatter<<<kGiantCtas, 256, 0, stream>>>(dr, root, direct, wlog, nwin, hp.ghist, hp.pairs);
    launches += 3;
    for (int w = 0; w < nwin; ++w) {
      const uint64_t approx = h.b / nwin + 1;  // grid sizing only
      const unsigned g = static_cast<unsigned>(std::max<uint64_t>(
          1, std::min<uint64_t>(static_cast<uint64_t>(ctx->sm_count) * 8, (approx + 256 * per - 1) / (256 * per))));
      k_giant_apply<<<g, 256, 0, stream>>>(dr, hp.pairs, wbeg, w, view_scratch(ctx, mode));
      ++launches;
    }
  }
  // head bitmaps tb of every heavy slice from the finished tables (grids per
  // size class: one (chunk, slice) grid sized for the longest slice of all
  // would launch mostly empty CTAs for the many short ones)
  for (const Cls& c : cls) {
    if (!c.cnt) continue;
    k_heavy_tb<<<dim3(gxc(c, c.mx / 16 + 1), c.cnt), 256, 0, stream>>>(d + c.r0, view_scratch(ctx, mode),
                                                                       ctx->heavy_flags + c.r0, hp.bits);
    ++launches;
  }
  for (size_t i = 0; i < hp.giant.size(); ++i) {
    const unsigned g = static_cast<unsigned>(std::max<uint64_t>(
        1, std::min<uint64_t>(static_cast<uint64_t>(ctx->sm_count) * 8, (hp.giant[i].b / 8 + 2047) / 2048)));
    k_heavy_tb<<<dim3(g, 1), 256, 0, stream>>>(d + n_reg + i, view_scratch(ctx, mode), ctx->heavy_flags + n_reg + i,
                                              hp.bits);
    ++launches;
  }
  for (const Cls& c : cls) {
    if (!c.cnt) continue;
    k_heavy_tail<<<dim3(gxc(c, (c.mx + 1) / 2 / kTailIlp), c.cnt), 256, 0, stream>>>(
        d + c.r0, view_scratch(ctx, mode), ctx->heavy_flags + c.r0, mask, hp.bits);
    k_heavy_head<<<dim3(gxc(c, (c.mx + 1) / 2 / 32 + 1), c.cnt), 256, 0, stream>>>(d + c.r0, ctx->heavy_flags + c.r0, mask,
                                                                          hp.bits);
    launches += 2;
  }
  for (size_t i = 0; i < hp.giant.size(); ++i) {  // one slice per launch: its bitmaps stay in L2
    const HeavyRow& h = hp.giant[i];
    const unsigned g = static_cast<unsigned>(std::max<uint64_t>(
        1, std::min<uint64_t>(static_cast<uint64_t>(ctx->sm_count) * 8, (h.n / 2 + 256 * per - 1) / (256 * per))));
    const uint32_t* tb = hp.bits + hp.bit_off[i];
    uint32_t* rb = hp.bits + hp.bit_off[i] + (static_cast<uint64_t>(h.b) + 31) / 32;
    k_heavy_tail_big<<<g, 256, 0, stream>>>(d + n_reg + i, view_scratch(ctx, mode), ctx->heavy_flags + n_reg + i, mask,
                                            tb, rb);
    const unsigned gh = static_cast<unsigned>(std::max<uint64_t>(
        1, std::min<uint64_t>(static_cast<uint64_t>(ctx->sm_count) * 8, (h.b / 32 + 255) / 256)));
    k_heavy_head_big<<<gh, 256, 0, stream>>>(d + n_reg + i, ctx->heavy_flags + n_reg + i, mask, rb);
    launches += 2;
  }
  k_heavy_exact<<<nh, 32, 0, stream>>>(d, view_scratch(ctx, mode), ctx->heavy_flags, mask, root, direct);
  NTCB_CUDA(cudaGetLastError());
  return launches;
}

void drop_heavy(ntcb_context* ctx) {
  if (!ctx->cache[kCacheHeavy]) return;
  for (auto& kv : ctx_cache<HeavyPlans>(ctx, kCacheHeavy)) {
    if (kv.second.rows) cudaFree(kv.second.rows);
    if (kv.second.bits) cudaFree(kv.second.bits);
    if (kv.second.pairs) cudaFree(kv.second.pairs);
    if (kv.second.ghist) cudaFree(kv.second.ghist);
  }
  ctx_cache_free<HeavyPlans>(ctx, kCacheHeavy);
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
  a.gscratch = view_scratch(ctx, mode);
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
