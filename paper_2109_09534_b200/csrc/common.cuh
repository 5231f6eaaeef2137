// Internal definitions shared by the ntc-b200 CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <vector>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "ntc_b200.h"

namespace ntcb {

// ---------------------------------------------------------------------------
// Errors.  Each C-ABI entry point catches these and maps them to the code of
// the exception the reference throws in the same situation.
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define NTCB_CUDA(call)                                                                  \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      ::ntcb::fail(NTCB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

// ---------------------------------------------------------------------------
// Splitmix64 stream, bit-identical to ntc::RngStream (rng.hpp:13-63).
// ---------------------------------------------------------------------------
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {  // rng.hpp:55-59
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t fork64(uint64_t s, uint64_t tag) {  // rng.hpp:18-20
  return mix64(s ^ (kGolden * (tag + 1)));
}

// floor(c * n) in double, clamped to n; c >= 1 -> n (nmc.cpp:36-40).
__host__ __device__ __forceinline__ uint64_t blocksize_for(double c, uint64_t n) {
  if (c >= 1.0) return n;
  const uint64_t b = static_cast<uint64_t>(floor(c * static_cast<double>(n)));
  return b > n ? n : b;
}

// ---------------------------------------------------------------------------
// Device-resident mode view: CSR over the rows of the mode-m unfolding.
// Structure-of-arrays so that a CTA streams a slice with fully coalesced
// (and 128-bit vectorisable) loads:
//   off[rows+1]           slice p = entries [off[p], off[p+1])
//   oth[k][nnz]           k-th non-mode coordinate (ascending mode order)
//   val[nnz]              fp32 value
// Entry order inside a slice is the reference's (mode_view.cpp:5-7):
// lexicographic in the remaining coordinates.
// ---------------------------------------------------------------------------
// view arrays are padded so a whole 128-entry batch (512 bytes, the update's
// bulk copy) starting at any 32-entry boundary <= nnz stays in bounds
constexpr uint64_t kViewPad = 160;

struct DeviceView {
  uint64_t rows = 0;
  uint64_t max_slice = 0;     // longest resident slice
  uint64_t* off = nullptr;
  // oth/val are indexed by ABSOLUTE view position e; when the context keeps
  // only a slab of rows (ntcb_view_keep_rows, multi-GPU shards) they point
  // a_lo elements before their allocation, which covers [a_lo, e_hi + pad)
  uint32_t* oth[NTCB_MAX_ORDER - 1] = {};
  float* val = nullptr;
  uint64_t* h_off = nullptr;  // host copy of the offsets (shard planning, blocksizes)
  uint64_t row_lo = 0, row_hi = 0;  // resident rows [row_lo, row_hi)
  uint64_t a_lo = 0;                // first allocated entry (row_lo's start rounded down to 32)
};

// Kernel-argument bundle describing the factor matrices.
struct FactorArgs {
  const float* U[NTCB_MAX_ORDER];  // factor m: dims[m] x ld, fp32
  int order;
  int mode;
  int rank;
  int ld;
};

// Launch statistics gathered when profiling is on.
struct Profile {
  bool on = false;
  cudaEvent_t ev[4096];
  int kind[2048];
  int n = 0;
  uint64_t launches = 0;
  uint64_t update_launches = 0;
  // the item kernel alone (k_update_tc / k_update, without the split-row finalisation): start/end pairs
  cudaEvent_t kev[1024];
  int kn = 0;
};

inline ntcb_tuning default_tuning() {
  ntcb_tuning t{};
  t.no_tc = 0;
  t.no_nat = 0;
  t.tc_p = 0;
  t.update_wpc = 4;
  t.short_row = 2048;
  t.side_sampler_ctas = 0;
  t.heavy_per = 8;
  t.heavy_win_log2 = 24;
  t.heavy_big_log2 = 24;
  t.host_threads = 0;
  t.update_ctas_per_sm = 0;
  t.update_carveout = -1;
  t.peer_fence = 1;
  t.graph = 0;
  t.nat_pad = -1;
  t.tiny_sampler = 1;
  t.item_order = 0;
  return t;
}

// Per-context caches of the translation units (launch plans keyed by mode,
// row range and c).  Owned by the context, so two contexts on two host
// threads never share a container; a context itself is not re-entrant.
enum CacheSlot { kCacheUpdate = 0, kCacheSample, kCacheHeavy, kCacheMetrics, kCacheSlots };

}  // namespace ntcb

// The opaque context behind ntcb_context*.
struct ntcb_context {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int sm_count = 148;

  // tensor
  int order = 0;
  uint64_t dims[NTCB_MAX_ORDER] = {};
  uint64_t nnz = 0;
  ntcb::DeviceView views[NTCB_MAX_ORDER];

  // factors
  uint64_t rank = 0;
  uint64_t ld = 0;
  bool nat_padded = false;  // 128-byte rows below rank 25: the update runs the NAT kernel
  float* A[NTCB_MAX_ORDER] = {};
  float* peerA[NTCB_MAX_ORDER][7] = {};  // replicas of A[m] on other GPUs (fused exchange)
  int n_peers[NTCB_MAX_ORDER] = {};
  std::vector<void*> ipc_opened;          // mappings to close at destroy
  float* Y[NTCB_MAX_ORDER] = {};

  // sampled-set masks, one bit per view entry, per (mode, inner-iteration parity)
  uint32_t* mask[NTCB_MAX_ORDER][2] = {};
  uint64_t mask_words = 0;
  int mask_parity[NTCB_MAX_ORDER] = {};
  cudaStream_t side = nullptr;  // sampler stream (sampling never reads factors)
  cudaEvent_t ev_sampled[NTCB_MAX_ORDER][2] = {};
  cudaEvent_t ev_consumed[NTCB_MAX_ORDER][2] = {};
  cudaEvent_t ev_side_done = nullptr;  // collect(): the main stream waits for the side stream
  bool consumed_valid[NTCB_MAX_ORDER][2] = {};
  float* partial = nullptr;  // split-row partial sums
  uint64_t partial_n = 0;
  uint32_t* perm_scratch = nullptr;  // per-entry Fisher-Yates scratch for slices too big for smem
  uint64_t perm_scratch_n = 0;
  int* heavy_flags = nullptr;  // per heavy slice: a draw may need Lemire rejection
  uint32_t heavy_flags_n = 0;
  unsigned long long* counters = nullptr;  // [1] first error key, [2],[3] update cursors, [4],[5] sampler cursors
  unsigned long long* h_counters = nullptr;  // pinned mirror
  double* red = nullptr;  // metrics partials
  uint64_t red_n = 0;
  int error_mode = -1;    // mode of the queued updates (error text)

  ntcb_tuning tune = ntcb::default_tuning();
  uint64_t plan_epoch = 0;              // bumped whenever cached launch plans are dropped
  void* cache[ntcb::kCacheSlots] = {};  // per-TU plan maps (see CacheSlot)
  void* host = nullptr;                 // capi.cu host bookkeeping (HostState)

  ntcb::Profile prof;
};

namespace ntcb {
// Profiling: an event on the library stream before / after the update's item kernel.
inline void prof_kernel_mark(ntcb_context* ctx) {
  Profile& pf = ctx->prof;
  if (!pf.on || pf.kn >= 1024) return;
  cudaEventRecord(pf.kev[pf.kn++], ctx->stream);
}
// The per-entry sampler scratch, indexed by absolute view position of `mode`.
inline uint32_t* view_scratch(ntcb_context* ctx, int mode) {
  return ctx->perm_scratch ? ctx->perm_scratch - ctx->views[mode].a_lo : nullptr;
}
// The map of cache slot k of a context, created on first use.
template <class M>
M& ctx_cache(ntcb_context* ctx, int k) {
  if (!ctx->cache[k]) ctx->cache[k] = new M();
  return *static_cast<M*>(ctx->cache[k]);
}
template <class M>
void ctx_cache_free(ntcb_context* ctx, int k) {
  delete static_cast<M*>(ctx->cache[k]);
  ctx->cache[k] = nullptr;
}
}  // namespace ntcb
