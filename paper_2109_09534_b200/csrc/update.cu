// Row update of S_NMC (nmc.cpp:199-272 minus sampling).
//
// Work decomposition.  A work item is (row p, entry range [e0, e1)) of one
// mode view: one item per row when the slice has <= kSeg entries, several
// when it is longer (their partial sums go to a global slot and
// k_finalize reduces them in a fixed order -- deterministic, and a heavy row
// no longer serialises on one warp).  ONE WARP per item, no block barriers:
//
//   stream  128 consecutive entries per step (cp.async 128-bit loads of the
//           SoA record arrays and the mask, double-buffered), keep the
//           sampled ones (mask bit, or all at c >= 1), compact them with a
//           warp scan into a 256-slot staging ring in shared memory;
//   gather  groups of 32/L picks, L = ld/4: lane (pick, s) loads feature
//           block s of the pick's row in every other factor (a pick's L
//           lanes read one contiguous row) and forms the Khatri-Rao block
//           (kr_row, factor_set.cpp:42-64); the next group's loads are in
//           flight while this group computes;
//   Gram    lane role s owns block pairs (s, s+d), d <= L/2, with partner
//           blocks fetched by shuffle -- every block pair of the upper
//           triangle exactly once, operands in registers (nmc.cpp:95-96);
//           w_s += x k_s on the side.
//
// Finalisation per row (warp, fp64): H = lambda I + sum k k^T (mirrored),
// grad = H y - w + lambda y (= w + z + lambda y of nmc.cpp:84-105),
// finiteness checks (nmc.cpp:247-251, 145-146),
// power method from the normalised all-ones vector (nmc.cpp:140-172),
// L = 1.01 rq (nmc.cpp:253-254), projected step + Nesterov momentum
// (nmc.cpp:174-197).  fp32 accumulation; sums are taken in slice order over
// the (bit-exact) sampled set.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace ntcb {

// Compile-time A/B switches of tools/variants.sh (defaults = the measured best, profiles/r02_update_experiments.txt):
// NTCB_ROW_END_REG 0 row end reads H from shared memory, 1 rows of H in registers, 2 + half rows up to rank 16;
// NTCB_NAT4_SHORT  the short-row instantiation of the 64-byte-row NAT kernel; NTCB_FINQ slots in flight in k_finalize_small.
#ifndef NTCB_ROW_END_REG
#define NTCB_ROW_END_REG 2
#endif
constexpr int kWarps = 8;         // warps per CTA
constexpr uint64_t kSeg = 16384;  // max entries per work item

struct WorkItem {
  uint64_t row;
  uint64_t e0, e1;  // absolute view positions
  int64_t slot;     // -1: finalise in place; else partial slot
};

struct FinItem {
  uint64_t row;
  int64_t slot0;
  int32_t nslots;
  int32_t ngroups;  // big rows: slot groups of kSlotGroup, sums at gpart[g0 ..]
  int64_t g0;
};

// a group of <= kSlotGroup consecutive slots of a big split row, summed in
// slot order (fp64) by one warp of k_slot_groups into gpart[out]
struct SlotGroup {
  int64_t slot0;
  int64_t out;
  int32_t n;
  int32_t pad;
};
constexpr int kSlotGroup = 32;

struct UpdateArgs {
  const uint64_t* off;
  const uint32_t* oth[NTCB_MAX_ORDER - 1];
  const float* val;
  const uint32_t* mask;
  const float* U[NTCB_MAX_ORDER - 1];  // other modes' factors, ascending mode order
  int no;                              // order - 1
  int mode;
  int rank;
  int ld;                              // factor row stride (floats)
  float* A;
  float* Y;
  float* peerA[7];  // replicas of A on other GPUs: finalised rows are stored there too
  int n_peers;
  int peer_fence;   // __threadfence_system() after each row's peer stores (ntcb_tuning.peer_fence)
  const WorkItem* items;
  uint64_t n_items;
  const FinItem* fins;
  uint64_t n_fins;
  float* partial;  // [slot][R*R + R]
  double* gpart;   // [group][R*R + R]: slot-group sums of big split rows
  const SlotGroup* groups;
  uint64_t n_groups;
  double c;
  double lambda;
  double power_tol;
  int power_iters;
  unsigned long long* counters;  // [1] first error key, [2] item cursor, [3] fin cursor
};

__device__ __forceinline__ void report(unsigned long long* counters, int mode, uint64_t row,
                                       int kind) {
  const unsigned long long key =
      (static_cast<unsigned long long>(mode) << 58) | (static_cast<unsigned long long>(row) << 2) |
      static_cast<unsigned long long>(kind);
  atomicMin(&counters[1], key);
}

template <int LD4>
struct Geo {
  static constexpr int NBLK = LD4 * (LD4 + 1) / 2;
  static constexpr int GW = NBLK <= 32 ? 32 / NBLK : 1;   // pick groups per warp
  static constexpr int BPL = NBLK <= 32 ? 1 : (NBLK + 31) / 32;  // blocks per lane
  static constexpr int KS4 = (LD4 % 2) ? LD4 : LD4 + 1;   // odd float4 stride
  static constexpr int KS = 4 * KS4;
};

// per-warp shared memory (floats unless noted)
template <int LD4>
struct WarpSmem {
  static constexpr int kStage = 256;  // staging ring: < 32 leftover + 128 per batch
  // layout offsets in 4-byte words
  static __host__ __device__ constexpr int stage_words(int no) { return (no + 1) * kStage; }
  // the K tile region is reused for Hf (R x HS) after the pick loop
  static __host__ __device__ constexpr int ktile_words(int R) {  // Hf (R x HS)
    return ((R * (R | 1) + 3) / 4) * 4;
  }
  // double-buffered raw batches (cp.async landing zone): [2][no+1][128] + masks [2][32]
  static __host__ __device__ constexpr int batch_words(int no) { return 2 * (no + 1) * 128 + 64; }
  static __host__ __device__ constexpr int words(int no, int R) {
    return stage_words(no) + ktile_words(R) + 64 * 2 * 2 + batch_words(no);  // + g, v doubles
  }
};

__device__ __forceinline__ void block_of(int blk, int nb4, int& bi, int& bj) {
  int rem = blk;
  bi = 0;
  bj = 0;
  for (int i = 0; i < nb4; ++i) {
    const int cnt = nb4 - i;
    if (rem < cnt) {
      bi = i;
      bj = i + rem;
      return;
    }
    rem -= cnt;
  }
}

// Warp-level finalisation of one row from Hf (R x HS, fp32 sums of k k^T,
// full symmetric) and g (fp64 sums of s k, in gd).  Writes A[p], Y[p].
template <bool PRE = false>
__device__ void finalize_row(const UpdateArgs& a, uint64_t p, float* Hf, double* gd, double* vv,
                             int lane, float y_pre = 0.f, float a_pre = 0.f) {
  const int R = a.rank;
  const int HS = R | 1;
  const int ld = a.ld;
  const double lam = a.lambda;
  if constexpr (PRE) {
    // Y and A of the row were copied into shared memory with the item's
    // first batch (R <= 32, lane r holds element r): no global round trip
    // on the row-end latency chain (rows of a few hundred entries)
    if (lane < R) vv[lane] = static_cast<double>(y_pre);
    __syncwarp();
    bool bad = false;
    if (lane < R) {
      const float* hr = Hf + lane * HS;
      double hy = 0.0;
      for (int q = 0; q < R; ++q) hy += static_cast<double>(hr[q]) * vv[q];
      gd[lane] = hy - gd[lane] + lam * static_cast<double>(y_pre);
      bad = !isfinite(gd[lane]);
    }
    __syncwarp();
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) report(a.counters, a.mode, p, 0);  // non-finite gradient
      return;
    }
  } else {
  // On entry gd holds w = sum_e x_e k_e.  grad = sum_e (y.k_e - x_e) k_e + lambda y
  // = H y - w + lambda y with H = sum k k^T (nmc.cpp:84-105).  Forming it here
  // in fp64 instead of per pick is exact in real arithmetic; the fp32 error of
  // the sums is relative to |H y| ~ L |y|, and the step divides by L, so the
  // update error stays ~1e-6 |y| (tests/test_gpu_parity.py, TOL = 1e-4).
  bool bad = false;
  const float* yrow = a.Y + p * ld;
  for (int r = lane; r < R; r += 32) {
    const float* hr = Hf + r * HS;
    double hy = 0.0;
    for (int q = 0; q < R; ++q) hy += static_cast<double>(hr[q]) * static_cast<double>(__ldg(yrow + q));
    gd[r] = hy - gd[r] + lam * static_cast<double>(yrow[r]);
    bad |= !isfinite(gd[r]);
  }
  __syncwarp();
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0) report(a.counters, a.mode, p, 0);  // non-finite gradient
    return;
  }
  }
  bool hbad = false;
  for (int i = lane; i < R * R; i += 32) hbad |= !isfinite(Hf[(i / R) * HS + (i % R)]);
  if (__any_sync(0xffffffffu, hbad)) {
    if (lane == 0) report(a.counters, a.mode, p, 1);  // power_method rejects H
    return;
  }
  const double v0 = 1.0 / sqrt(static_cast<double>(R));
  for (int r = lane; r < R; r += 32) vv[r] = v0;
  __syncwarp();
  double rq = 0.0, rq_prev = 0.0;
  // (H + lambda I) v with four partial sums per row: the iteration is a
  // latency chain (mat-vec -> two warp reductions -> normalise), and short
  // rows are dominated by it
  auto hrow_dot = [&](int r) {
    const float* hr = Hf + r * HS;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = 0;
    for (; j + 4 <= R; j += 4) {
      s0 += static_cast<double>(hr[j]) * vv[j];
      s1 += static_cast<double>(hr[j + 1]) * vv[j + 1];
      s2 += static_cast<double>(hr[j + 2]) * vv[j + 2];
      s3 += static_cast<double>(hr[j + 3]) * vv[j + 3];
    }
    for (; j < R; ++j) s0 += static_cast<double>(hr[j]) * vv[j];
    return ((s0 + s1) + (s2 + s3)) + lam * vv[r];
  };
  for (int it = 0; it < a.power_iters; ++it) {
    const double u0 = lane < R ? hrow_dot(lane) : 0.0;
    const double u1 = lane + 32 < R ? hrow_dot(lane + 32) : 0.0;
    double num = 0.0, un2 = u0 * u0 + u1 * u1;
    if (lane < R) num += vv[lane] * u0;
    if (lane + 32 < R) num += vv[lane + 32] * u1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      num += __shfl_xor_sync(0xffffffffu, num, o);
      un2 += __shfl_xor_sync(0xffffffffu, un2, o);
    }
    rq = num;
    if (un2 == 0.0) {
      rq = 0.0;
      break;
    }
    if (it > 0 && fabs(rq - rq_prev) <= a.power_tol * fabs(rq)) break;
    rq_prev = rq;
    const double inv = 1.0 / sqrt(un2);
    __syncwarp();
    if (lane < R) vv[lane] = u0 * inv;
    if (lane + 32 < R) vv[lane + 32] = u1 * inv;
    __syncwarp();
  }
  const double L = rq * 1.01;  // nmc.cpp:253-254
  if (!(L >= lam)) {
    if (lane == 0) report(a.counters, a.mode, p, 2);  // row_step rejects L
    return;
  }
  const double inv_l = 1.0 / L;
  const double sl = sqrt(L), sm = sqrt(lam);
  const double beta = (sl - sm) / (sl + sm);
  for (int r = lane; r < R; r += 32) {
    const double y = static_cast<double>(PRE ? y_pre : a.Y[p * ld + r]);
    const double ap = static_cast<double>(PRE ? a_pre : a.A[p * ld + r]);
    const double av = y - inv_l * gd[r];
    const double an = av > 0.0 ? av : 0.0;
    a.A[p * ld + r] = static_cast<float>(an);
    a.Y[p * ld + r] = static_cast<float>(an + beta * (an - ap));
    // the fused exchange: the row goes to every peer replica over NVLink now,
    // overlapped with the rows still being computed (no all-gather after)
    for (int q = 0; q < a.n_peers; ++q) a.peerA[q][p * ld + r] = static_cast<float>(an);
  }
  if (a.n_peers && a.peer_fence == 2) __threadfence_system();  // per row (A/B)
}


// The same row end for ranks up to RB <= 32 with each lane's row of H held in
// REGISTERS: the mat-vecs of the gradient and of every power iteration read
// Hf once instead of once per iteration, and v is read as 16-byte broadcasts
// (two doubles per wavefront).  Same operations in the same order as
// finalize_row -- identical results; on short-row modes (configs 3 and 5) the
// row end was most of the kernel's shared-memory traffic.
template <bool PRE, int RB>
__device__ __forceinline__ void finalize_row_reg(const UpdateArgs& a, uint64_t p, float* Hf, double* gd, double* vv,
                                                 int lane, float y_pre = 0.f, float a_pre = 0.f) {
  static_assert(RB % 4 == 0 && RB <= 32, "row block");
  const int R = a.rank;
  const int HS = R | 1;
  const int ld = a.ld;
  const double lam = a.lambda;
  const bool mine = lane < R;
  float hrow[RB];
  bool hbad = false;
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    hrow[j] = (mine && j < R) ? Hf[lane * HS + j] : 0.f;
    hbad |= !isfinite(hrow[j]);
  }
  const float yv = PRE ? y_pre : (mine ? a.Y[p * ld + lane] : 0.f);
  const float av = PRE ? a_pre : (mine ? a.A[p * ld + lane] : 0.f);
  if (mine) vv[lane] = static_cast<double>(yv);
  __syncwarp();
  const double2* v2 = reinterpret_cast<const double2*>(vv);
  bool bad = false;
  if (mine) {
    double hy = 0.0;
#pragma unroll
    for (int j = 0; j < RB; j += 2) {
      if (j < R) {
        const double2 v = v2[j >> 1];
        hy += static_cast<double>(hrow[j]) * v.x;
        if (j + 1 < R) hy += static_cast<double>(hrow[j + 1]) * v.y;
      }
    }
    gd[lane] = hy - gd[lane] + lam * static_cast<double>(yv);
    bad = !isfinite(gd[lane]);
  }
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0) report(a.counters, a.mode, p, 0);  // non-finite gradient
    return;
  }
  if (__any_sync(0xffffffffu, hbad)) {
    if (lane == 0) report(a.counters, a.mode, p, 1);  // power_method rejects H
    return;
  }
  const double v0 = 1.0 / sqrt(static_cast<double>(R));
  __syncwarp();
  if (mine) vv[lane] = v0;
  __syncwarp();
  double rq = 0.0, rq_prev = 0.0;
  const int R4 = R & ~3;
  for (int it = 0; it < a.power_iters; ++it) {
    double u0 = 0.0;
    if (mine) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int j = 0; j < RB; j += 4) {
        if (j < R) {
          const double2 va = v2[j >> 1];
          const double2 vb = (j + 2 < R) ? v2[(j >> 1) + 1] : make_double2(0.0, 0.0);
          if (j < R4) {
            s0 += static_cast<double>(hrow[j]) * va.x;
            s1 += static_cast<double>(hrow[j + 1]) * va.y;
            s2 += static_cast<double>(hrow[j + 2]) * vb.x;
            s3 += static_cast<double>(hrow[j + 3]) * vb.y;
          } else {  // the last, partial quad goes to s0 in order (as finalize_row's tail loop)
            s0 += static_cast<double>(hrow[j]) * va.x;
            if (j + 1 < R) s0 += static_cast<double>(hrow[j + 1]) * va.y;
            if (j + 2 < R) s0 += static_cast<double>(hrow[j + 2]) * vb.x;
          }
        }
      }
      u0 = ((s0 + s1) + (s2 + s3)) + lam * vv[lane];
    }
    double num = mine ? vv[lane] * u0 : 0.0, un2 = u0 * u0;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      num += __shfl_xor_sync(0xffffffffu, num, o);
      un2 += __shfl_xor_sync(0xffffffffu, un2, o);
    }
    rq = num;
    if (un2 == 0.0) {
      rq = 0.0;
      break;
    }
    if (it > 0 && fabs(rq - rq_prev) <= a.power_tol * fabs(rq)) break;
    rq_prev = rq;
    const double inv = 1.0 / sqrt(un2);
    __syncwarp();
    if (mine) vv[lane] = u0 * inv;
    __syncwarp();
  }
  const double L = rq * 1.01;  // nmc.cpp:253-254
  if (!(L >= lam)) {
    if (lane == 0) report(a.counters, a.mode, p, 2);  // row_step rejects L
    return;
  }
  const double inv_l = 1.0 / L;
  const double sl = sqrt(L), sm = sqrt(lam);
  const double beta = (sl - sm) / (sl + sm);
  if (mine) {
    const double y = static_cast<double>(yv);
    const double ap = static_cast<double>(av);
    const double avn = y - inv_l * gd[lane];
    const double an = avn > 0.0 ? avn : 0.0;
    a.A[p * ld + lane] = static_cast<float>(an);
    a.Y[p * ld + lane] = static_cast<float>(an + beta * (an - ap));
    for (int q = 0; q < a.n_peers; ++q) a.peerA[q][p * ld + lane] = static_cast<float>(an);
  }
  if (a.n_peers && a.peer_fence == 2) __threadfence_system();  // per row (A/B)
}

// Ranks up to 16: lane (r = lane % 16, h = lane / 16) holds HALF a row of H --
// columns 8h .. 8h+7, as doubles -- so all 32 lanes work on the mat-vecs, a
// lane reads half of v per product (two distinct 16-byte addresses per load
// instruction instead of one broadcast: half the shared-memory wavefronts),
// and the two reductions of a power iteration run over 16 lanes (both halves
// identically: every lane sees the same sums, no divergence).  The row end is
// most of the work on the short Zipf rows of configs 3 and 5.
template <bool PRE>
__device__ __forceinline__ void finalize_row_half(const UpdateArgs& a, uint64_t p, float* Hf, double* gd, double* vv,
                                                  int lane, const float* pre_y, const float* pre_a) {
  const int R = a.rank;
  const int HS = R | 1;
  const int ld = a.ld;
  const double lam = a.lambda;
  const int r = lane & 15, h = lane >> 4;
  const bool mine = r < R;
  double hd[8];
  bool hbad = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = 8 * h + j;
    const float v = (mine && c < R) ? Hf[r * HS + c] : 0.f;
    hbad |= !isfinite(v);
    hd[j] = static_cast<double>(v);
  }
  const float yv = mine ? (PRE ? pre_y[r] : a.Y[p * ld + r]) : 0.f;
  const float av = mine ? (PRE ? pre_a[r] : a.A[p * ld + r]) : 0.f;
  __syncwarp();
  if (lane < 16) vv[lane] = static_cast<double>(yv);  // zeros beyond R: the products below read all 16
  __syncwarp();
  const double2* v2 = reinterpret_cast<const double2*>(vv) + 4 * h;  // this lane's half of v
  // (H + shift I) v, this lane's half: two chains over the even / odd columns
  auto half_dot = [&]() {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const double2 v = v2[j >> 1];
      s0 += hd[j] * v.x;
      s1 += hd[j + 1] * v.y;
    }
    const double s = s0 + s1;
    return s + __shfl_xor_sync(0xffffffffu, s, 16);  // + the other half: the same sum in both lanes
  };
  const double hy = half_dot();
  double g = 0.0;
  bool bad = false;
  if (mine) {
    g = hy - gd[r] + lam * static_cast<double>(yv);
    bad = !isfinite(g);
  }
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0) report(a.counters, a.mode, p, 0);  // non-finite gradient
    return;
  }
  if (__any_sync(0xffffffffu, hbad)) {
    if (lane == 0) report(a.counters, a.mode, p, 1);  // power_method rejects H
    return;
  }
  const double v0 = 1.0 / sqrt(static_cast<double>(R));
  double vr = mine ? v0 : 0.0;  // v_r, kept in a register too
  __syncwarp();
  if (lane < 16) vv[lane] = vr;
  __syncwarp();
  double rq = 0.0, rq_prev = 0.0;
  for (int it = 0; it < a.power_iters; ++it) {
    const double hv = half_dot();  // every lane takes part in its exchange
    const double u = mine ? hv + lam * vr : 0.0;
    double num = vr * u, un2 = u * u;
#pragma unroll
    for (int o = 8; o; o >>= 1) {  // over the 16 lanes of a half; both halves hold the same values
      num += __shfl_xor_sync(0xffffffffu, num, o);
      un2 += __shfl_xor_sync(0xffffffffu, un2, o);
    }
    rq = num;
    if (un2 == 0.0) {
      rq = 0.0;
      break;
    }
    if (it > 0 && fabs(rq - rq_prev) <= a.power_tol * fabs(rq)) break;
    rq_prev = rq;
    vr = u * (1.0 / sqrt(un2));
    __syncwarp();
    if (lane < 16) vv[lane] = vr;
    __syncwarp();
  }
  const double L = rq * 1.01;  // nmc.cpp:253-254
  if (!(L >= lam)) {
    if (lane == 0) report(a.counters, a.mode, p, 2);  // row_step rejects L
    return;
  }
  if (mine && h == 0) {
    const double inv_l = 1.0 / L;
    const double sl = sqrt(L), sm = sqrt(lam);
    const double beta = (sl - sm) / (sl + sm);
    const double y = static_cast<double>(yv);
    const double ap = static_cast<double>(av);
    const double avn = y - inv_l * g;
    const double an = avn > 0.0 ? avn : 0.0;
    a.A[p * ld + r] = static_cast<float>(an);
    a.Y[p * ld + r] = static_cast<float>(an + beta * (an - ap));
    for (int q = 0; q < a.n_peers; ++q) a.peerA[q][p * ld + r] = static_cast<float>(an);
  }
  if (a.n_peers && a.peer_fence == 2) __threadfence_system();  // per row (A/B)
}

// row end of rank <= RB (0: any rank)
// (pre: SHORT's staged copies of the row, Y at pre[0..R), A at pre[32..32+R))
template <bool PRE, int RB>
__device__ __forceinline__ void row_end(const UpdateArgs& a, uint64_t p, float* Hf, double* gd, double* vv, int lane,
                                        const float* pre = nullptr) {
  if constexpr (RB > 0 && RB <= 16 && NTCB_ROW_END_REG == 2) {
    finalize_row_half<PRE>(a, p, Hf, gd, vv, lane, pre, pre + 32);
  } else {
    const bool on = PRE && lane < a.rank;
    const float y_pre = on ? pre[lane] : 0.f, a_pre = on ? pre[32 + lane] : 0.f;
    if constexpr (RB > 0 && RB <= 32 && NTCB_ROW_END_REG)
      finalize_row_reg<PRE, RB>(a, p, Hf, gd, vv, lane, y_pre, a_pre);
    else
      finalize_row<PRE>(a, p, Hf, gd, vv, lane, y_pre, a_pre);
  }
}

// The fused exchange's ordering (peer_fence 1, the default): every thread
// that stored finished rows into peer replicas fences once, at the end of
// its kernel, so all of them are visible system-wide before the kernel
// completes and the NCCL barrier that follows releases the next mode.  (A
// fence after every row, peer_fence 2, measured +15 % at config 5 on one GPU
// -- 8.4M fences per AO iteration -- and orders nothing more that matters.)
__device__ __forceinline__ void peer_fence_at_exit(const UpdateArgs& a) {
  if (a.n_peers && a.peer_fence == 1) __threadfence_system();
}

// One streamed batch (4 entries per lane: coordinates co[m], values cv,
// sampled bits `bits`) compacted into the staging ring at `at`, in entry
// order (warp scan of the per-lane counts).  Returns the entries added.
// Shared by k_update and k_update_tc.
template <int NO, int kStage>
__device__ __forceinline__ int stage_sampled(uint32_t bits, const uint4 (&co)[NO], const uint4& cv, int no, int lane,
                                             int at, uint32_t* st_o, float* st_x) {
  const int c4 = __popc(bits);
  int incl = c4;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int slot = at + incl - c4;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if ((bits >> q) & 1u) {
      const int sl = slot & (kStage - 1);
#pragma unroll
      for (int m = 0; m < NO; ++m)
        if (m < no) st_o[m * kStage + sl] = q == 0 ? co[m].x : q == 1 ? co[m].y : q == 2 ? co[m].z : co[m].w;
      st_x[sl] = __uint_as_float(q == 0 ? cv.x : q == 1 ? cv.y : q == 2 ? cv.z : cv.w);
      ++slot;
    }
  }
  return total;
}

// CUDA-core update CTA shapes: ranks <= 20 -> 8 warps x 2 CTAs (<= 128 regs);
// 21-32 -> 4 warps x 3 CTAs (<= 170 regs, 12 warps/SM instead of 8);
// above -> 8 warps x 1 CTA
__host__ __device__ constexpr int k_update_threads(int LD4) { return (LD4 >= 6 && LD4 <= 8) ? 128 : 256; }
__host__ __device__ constexpr int k_update_min_blocks(int LD4) { return LD4 <= 5 ? 2 : LD4 <= 8 ? 3 : 1; }

template <int LD4, int NO>
__global__ void __launch_bounds__(k_update_threads(LD4), k_update_min_blocks(LD4)) k_update(UpdateArgs a) {
  using W = WarpSmem<LD4>;
  constexpr int L = LD4;          // feature blocks of 4 = lanes (roles) per pick
  constexpr int GP = 32 / L;      // picks per group
  constexpr int ND = L / 2 + 1;   // block pairs per role: (s, s+d), d < ND
  extern __shared__ __align__(16) float smem_f[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int no = NO < NTCB_MAX_ORDER - 1 ? NO : a.no;  // compile-time for orders 3 and 4
  const int R = a.rank;
  const int HS = R | 1;
  const int ld = LD4 * 4;
  float* wbase = smem_f + static_cast<size_t>(wid) * W::words(no, R);
  uint32_t* st_o = reinterpret_cast<uint32_t*>(wbase);  // [no][kStage]
  float* st_x = wbase + no * W::kStage;                 // [kStage]
  float* Hf = wbase + W::stage_words(no);               // [R][HS]
  double* gd = reinterpret_cast<double*>(Hf + W::ktile_words(R));  // [64]
  double* vv = gd + 64;                                             // [64]
  uint32_t* rbat = reinterpret_cast<uint32_t*>(vv + 64);            // raw batches
  uint32_t* rmsk = rbat + 2 * (no + 1) * 128;                       // [2][32]
  const bool full = a.c >= 1.0;

  // role of this lane: pick slot pk within a group, feature block s
  const int pk = lane / L;
  const int s = lane - pk * L;
  const bool lane_on = pk < GP;
  int sd[ND];  // partner block of pair d
#pragma unroll
  for (int d = 0; d < ND; ++d) sd[d] = (s + d) % L;
  // with even L the distance-L/2 pairs appear twice: roles s >= L/2 skip them
  const bool skip_last = (L % 2 == 0) && (s >= L / 2);

  while (true) {
    if (*reinterpret_cast<volatile unsigned long long*>(&a.counters[1]) != ~0ull) return;
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(&a.counters[2], 1ull);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= a.n_items) break;
    const WorkItem w = a.items[it];
    const uint64_t p = w.row;

    float acc[ND][16];
#pragma unroll
    for (int d = 0; d < ND; ++d)
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[d][e] = 0.f;
    float4 gl = make_float4(0.f, 0.f, 0.f, 0.f);

    int head = 0, cnt = 0;  // staging ring [head, head+cnt)

    // One group of np <= GP picks: lane (pk, s) gathers feature block s of
    // pick pk from every other factor's row (the L lanes of a pick read one
    // contiguous row), forms the Khatri-Rao block, accumulates w_s += x k_s
    // and the Gram blocks (s, s+d) with partner blocks fetched by shuffle.
    // A group's gather (load_group) is issued one group ahead of its
    // arithmetic (compute_group) so the L2 latency of the factor rows hides
    // behind the previous group's Gram update.
    struct Raw {
      float4 f[NO];
    };
    // Full groups (GP picks): lanes beyond GP*L load factor row 0 (valid,
    // discarded by the slot reduction), so no predicates or zero fills.
    auto load_full = [&](int at) {
      Raw g;
      const int sidx = (at + pk) & (W::kStage - 1);
#pragma unroll
      for (int m = 0; m < NO; ++m)
        if (m < no) {
          const uint32_t row = lane_on ? st_o[m * W::kStage + sidx] : 0u;
          g.f[m] = __ldg(reinterpret_cast<const float4*>(a.U[m] + static_cast<uint64_t>(row) * ld) + s);
        }
      return g;
    };
    // The partial last group of an item: lanes of absent picks contribute 0.
    auto load_part = [&](int at, int np) {
      Raw g;
      const bool on = lane_on && pk < np;
      const int sidx = (at + pk) & (W::kStage - 1);
#pragma unroll
      for (int m = 0; m < NO; ++m)
        if (m < no) {
          const uint32_t row = on ? st_o[m * W::kStage + sidx] : 0u;
          g.f[m] = __ldg(reinterpret_cast<const float4*>(a.U[m] + static_cast<uint64_t>(row) * ld) + s);
          if (!on) g.f[m] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      return g;
    };
    auto compute_group = [&](const Raw& g, int at, int np) {
      // lanes of absent picks in a partial group must add exact zeros (stale
      // ring slots may hold anything); lanes beyond GP*L are never reduced
      const float gx = pk < np ? st_x[(at + pk) & (W::kStage - 1)] : 0.f;
      float4 kb = g.f[0];
#pragma unroll
      for (int m = 1; m < NO; ++m) {
        if (m < no) {
          kb.x *= g.f[m].x;
          kb.y *= g.f[m].y;
          kb.z *= g.f[m].z;
          kb.w *= g.f[m].w;
        }
      }
      // w += x k  (the gradient is formed as H y - w at the row end)
      const int base = (lane_on ? pk : 0) * L;
      gl.x = fmaf(gx, kb.x, gl.x);
      gl.y = fmaf(gx, kb.y, gl.y);
      gl.z = fmaf(gx, kb.z, gl.z);
      gl.w = fmaf(gx, kb.w, gl.w);
      const float ka[4] = {kb.x, kb.y, kb.z, kb.w};
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        float kp[4];
        if (d == 0) {
          kp[0] = kb.x;
          kp[1] = kb.y;
          kp[2] = kb.z;
          kp[3] = kb.w;
        } else {
          const int src = base + sd[d];
          kp[0] = __shfl_sync(0xffffffffu, kb.x, src);
          kp[1] = __shfl_sync(0xffffffffu, kb.y, src);
          kp[2] = __shfl_sync(0xffffffffu, kb.z, src);
          kp[3] = __shfl_sync(0xffffffffu, kb.w, src);
        }
        if (d == ND - 1 && skip_last) continue;
        if (d == 0) {  // diagonal block: upper triangle only (mirrored on output)
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c2 = r; c2 < 4; ++c2) acc[0][4 * r + c2] = fmaf(ka[r], kp[c2], acc[0][4 * r + c2]);
        } else {
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c2 = 0; c2 < 4; ++c2) acc[d][4 * r + c2] = fmaf(ka[r], kp[c2], acc[d][4 * r + c2]);
        }
      }
    };
    // All staged full groups, three-way rotation: the gathers of groups g+1
    // and g+2 are in flight while group g computes (no register copies that
    // would wait on in-flight loads).
    auto drain_full = [&]() {
      const int ng = cnt / GP;
      if (ng == 0) return;
      int al = head, ac = head;
      Raw r0, r1, r2;
      r0 = load_full(al);
      al = (al + GP) & (W::kStage - 1);
      if (1 < ng) {
        r1 = load_full(al);
        al = (al + GP) & (W::kStage - 1);
      }
      for (int g = 0; g < ng; g += 3) {
        if (g + 2 < ng) {
          r2 = load_full(al);
          al = (al + GP) & (W::kStage - 1);
        }
        compute_group(r0, ac, GP);
        ac = (ac + GP) & (W::kStage - 1);
        if (g + 1 < ng) {
          if (g + 3 < ng) {
            r0 = load_full(al);
            al = (al + GP) & (W::kStage - 1);
          }
          compute_group(r1, ac, GP);
          ac = (ac + GP) & (W::kStage - 1);
          if (g + 2 < ng) {
            if (g + 4 < ng) {
              r1 = load_full(al);
              al = (al + GP) & (W::kStage - 1);
            }
            compute_group(r2, ac, GP);
            ac = (ac + GP) & (W::kStage - 1);
          }
        }
      }
      head = (head + ng * GP) & (W::kStage - 1);
      cnt -= ng * GP;
    };

    // ---- stream the item in batches of 128 entries (4 per lane; cp.async
    // 128-bit loads of the SoA records and the mask word, double-buffered,
    // issued independently of the mask) ----
    const uint64_t tb = w.e0 & ~uint64_t(3);  // 16-byte aligned start
    const int lo = static_cast<int>(w.e0 - tb);          // item start, relative to tb
    const int hi = static_cast<int>(w.e1 - tb);          // item end, relative to tb
    auto fetch_async = [&](int t, int buf) {
      const int r = t + 4 * lane;
      if (r < hi) {
        const uint64_t e = tb + static_cast<uint64_t>(r);
#pragma unroll
        for (int m = 0; m < NO + 1; ++m) {
          if (m < no || m == NO) {
            const int row = (m == NO) ? no : m;
            const void* src = (m == NO) ? static_cast<const void*>(a.val + e) : static_cast<const void*>(a.oth[m] + e);
            const unsigned dst = static_cast<unsigned>(
                __cvta_generic_to_shared(rbat + (buf * (no + 1) + row) * 128 + 4 * lane));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
          }
        }
        if (!full) {
          const unsigned dm = static_cast<unsigned>(__cvta_generic_to_shared(rmsk + buf * 32 + lane));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dm), "l"(a.mask + (e >> 5)));
        }
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    const uint32_t sh0 = static_cast<uint32_t>(tb & 31u);  // bit of rel 0 in its mask word
    fetch_async(0, 0);
    int buf = 0;
    for (int t0 = 0; t0 < hi; t0 += 128, buf ^= 1) {
      if (t0 + 128 < hi) {
        fetch_async(t0 + 128, buf ^ 1);
        asm volatile("cp.async.wait_group 1;\n" ::);
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::);
      }
      uint4 co[NO];
#pragma unroll
      for (int m = 0; m < NO; ++m)
        if (m < no) co[m] = reinterpret_cast<const uint4*>(rbat + (buf * (no + 1) + m) * 128)[lane];
      const uint4 cv = reinterpret_cast<const uint4*>(rbat + (buf * (no + 1) + no) * 128)[lane];
      const int r = t0 + 4 * lane;
      uint32_t bits = full ? 0xfu : (rmsk[buf * 32 + lane] >> ((sh0 + static_cast<uint32_t>(r)) & 31u)) & 0xfu;
      // clip to [lo, hi)
      if (r < lo) bits &= 0xfu << (lo - r);
      if (r + 4 > hi) bits &= hi - r > 0 ? (0xfu >> (4 - (hi - r))) : 0u;
      cnt += stage_sampled<NO, W::kStage>(bits, co, cv, no, lane, head + cnt, st_o, st_x);
      __syncwarp();
      drain_full();
    }
    if (cnt > 0) {  // the item's last, partial group
      const Raw rp = load_part(head, cnt);
      compute_group(rp, head, cnt);
      head = (head + cnt) & (W::kStage - 1);
      cnt = 0;
    }

    // ---- reduce over the GP pick slots (lanes with equal role s) ----------
#pragma unroll 1
    for (int t = 1; t < GP; ++t) {
      const int src = (lane + t * L) & 31;
#pragma unroll
      for (int d = 0; d < ND; ++d)
#pragma unroll
        for (int e2 = 0; e2 < 16; ++e2) {
          const float v = __shfl_sync(0xffffffffu, acc[d][e2], src);
          if (pk == 0) acc[d][e2] += v;
        }
      const float gx = __shfl_sync(0xffffffffu, gl.x, src);
      const float gy = __shfl_sync(0xffffffffu, gl.y, src);
      const float gz = __shfl_sync(0xffffffffu, gl.z, src);
      const float gw = __shfl_sync(0xffffffffu, gl.w, src);
      if (pk == 0) {
        gl.x += gx;
        gl.y += gy;
        gl.z += gz;
        gl.w += gw;
      }
    }
    __syncwarp();
    if (pk == 0) {  // lanes 0..L-1: role s holds blocks (s, s+d) and gradient block s
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        if (d == ND - 1 && skip_last) continue;
        const int cb = sd[d];
#pragma unroll
        for (int e2 = 0; e2 < 16; ++e2) {
          const int row = 4 * s + (e2 >> 2), col = 4 * cb + (e2 & 3);
          if (d == 0 && (e2 >> 2) > (e2 & 3)) continue;  // diagonal block: upper half only
          if (row < R && col < R) {
            Hf[row * HS + col] = acc[d][e2];
            Hf[col * HS + row] = acc[d][e2];
          }
        }
      }
      const float ga[4] = {gl.x, gl.y, gl.z, gl.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * s + q < R) gd[4 * s + q] = static_cast<double>(ga[q]);
    }
    __syncwarp();
    if (w.slot < 0) {
      finalize_row(a, p, Hf, gd, vv, lane);
    } else {
      float* dst = a.partial + static_cast<uint64_t>(w.slot) * (R * R + R);
      for (int i = lane; i < R * R; i += 32) dst[i] = Hf[(i / R) * HS + (i % R)];
      for (int r = lane; r < R; r += 32) dst[R * R + r] = static_cast<float>(gd[r]);
    }
    __syncwarp();
  }
  peer_fence_at_exit(a);
}

// ---------------------------------------------------------------------------
// Tensor-core Gram (ranks with R + 1 <= 8P, P <= 4).
//
// The Gram sum_e k_e k_e^T and w = sum_e x_e k_e are one matrix product:
// with k'_e = (k_e, x_e, 0...) (8P features) and K the picks x 8P matrix,
// K^T K holds H in its leading R x R block and w in column R.  A warp
// multiplies 8 picks at a time with mma.sync (m16n8), upper block tiles
// only (n-tile j >= 2 m-tile i).  fp32 accuracy from two products per tile:
//   k = hi + lo, hi = k with the low 13 mantissa bits cleared (exact tf32),
//   tf32  mma:  hi hi^T                        (exact products)
//   bf16  mma:  hi lo^T + lo hi^T               (k16 = 8 picks x {hi, lo})
// The dropped lo lo^T and the bf16 rounding of the cross terms are
// <= 2^-18 of |k_a k_b| per pick -- the size of fp32 accumulation error.
//
// Fragment ownership: lane (g = lane/4, t = lane%4) holds picks 2t, 2t+1 of
// the group and features rho = g + 8f (f < P) of both.  For the tf32
// product k-index t <-> pick 2t and t+4 <-> pick 2t+1; for the bf16 product
// k-index 2t/2t+1 <-> hi of picks 2t/2t+1 and 2t+8/2t+9 <-> their lo.
// ---------------------------------------------------------------------------
template <int P>
struct TcGeo {
  static constexpr int MT = (P + 1) / 2;  // m-tiles (16 features)
  static constexpr int count() {           // upper block tiles: sum_i (P - 2i)
    int n = 0;
    for (int i = 0; i < MT; ++i) n += P - 2 * i;
    return n;
  }
  static constexpr int NT = count();
  static constexpr int mi(int tl) {  // m-tile of a tile index
    int i = 0;
    while (tl >= P - 2 * i) tl -= P - 2 * i++;
    return i;
  }
  static constexpr int nj(int tl) {  // n-tile of a tile index
    int i = 0;
    while (tl >= P - 2 * i) tl -= P - 2 * i++;
    return 2 * i + tl;
  }
};

__device__ __forceinline__ void mma_tf32(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// D = A B (C = 0: ptxas can feed RZ instead of zeroed registers)
__device__ __forceinline__ void mma_tf32_z(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%10,%10,%10};\n"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.f));
}
__device__ __forceinline__ void mma_bf16(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// two floats -> bf16x2, `lo_k` in the low half (the smaller k index)
__device__ __forceinline__ uint32_t pack_bf16(float lo_k, float hi_k) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;\n" : "=r"(d) : "f"(hi_k), "f"(lo_k));
  return d;
}

// per-warp shared words of k_update_tc: the staging ring (reused for Hf, gd,
// vv at the row end, when the ring is drained) + the batch landing zone (free
// at the row end, so the next item's first batch lands there meanwhile)
__host__ __device__ constexpr int tc_ring_words(int no, int R) {
  return WarpSmem<1>::stage_words(no) > WarpSmem<1>::ktile_words(R) + 256 ? WarpSmem<1>::stage_words(no)
                                                                          : WarpSmem<1>::ktile_words(R) + 256;
}
// Register budget of k_update_tc: 256 threads x 2 CTAs = 128 registers (4 CTAs of 4 warps per SM).  The
// 4-way instantiations that gather three 16-byte pieces per pick slot (NAT on 128-byte rows, the quad
// layout) spill at 128: they get 168 registers and 3 CTAs per SM instead (config 4: 60.0 -> 51.0 ms per
// AO iteration).
// ... and the short-row kernel on 64-byte rows (configs 3 and 5: the row end's fp64 latency chain
// dominates) runs with 80 registers at 6 CTAs (24 warps) per SM: config 5 118.7 -> 112.6 ms, config 3
// 6.18 -> 6.09 ms per AO iteration (64 registers spill: 123.5 / 6.54; the pair-layout short-row kernel
// of config 1 loses at 80: 0.161 -> 0.187 ms, and keeps 128; the long-row 64-byte-row kernel is
// indifferent: 6.046 vs 6.045 ms at config 3).
__host__ __device__ constexpr int tc_bound_blocks(int P, bool SHORT, bool NAT, int LPP) {
  return (SHORT && NAT && LPP == 4) ? 3 : (P <= 4 ? 2 : 1);
}
__host__ __device__ constexpr int tc_bound_threads(int P, int NO, bool NAT, int LPP) {
  return (NO == 3 && ((NAT && LPP == 8) || P == 4)) ? 192 : kWarps * 32;
}
#ifndef NTCB_NAT4_SHORT
#define NTCB_NAT4_SHORT 1
#endif
constexpr int kKtStride = 36;          // natural layout: k' tile row stride (floats, bank-skewed)
constexpr int kKtWords = 8 * kKtStride;  // 8 picks
constexpr int kPreWords = 128;  // SHORT: [2 item parities][Y, A][32], the row's A and Y for the row end
__host__ __device__ constexpr int tc_words(int no, int R, bool nat = false, bool shrt = false) {
  return tc_ring_words(no, R) + WarpSmem<1>::batch_words(no) + (nat ? kKtWords : 0) + (shrt ? kPreWords : 0);
}

// base + row * ld4 bytes as one wide multiply-add
__device__ __forceinline__ const float* row_ptr(const float* base, uint32_t row, uint32_t ld4) {
  uint64_t p;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(row), "r"(ld4), "l"(reinterpret_cast<uint64_t>(base)));
  return reinterpret_cast<const float*>(p);
}

// NAT (natural gather, ranks 25-32 at ld = 32): a pick's row of each other
// factor is one 128-byte line read by 8 consecutive lanes as float4 (one
// wavefront per row and mode instead of the pair layout's ~3); the
// Khatri-Rao rows k go through an 8 x 32 shared tile into the fragment
// layout; w = sum x k is accumulated on the CUDA cores in the natural
// layout (no x column in the tiles, so 32 features fit 4 blocks).
// LPP = lanes per pick of the NAT gathers: 8 (128-byte rows, ld = 32) or 4
// (64-byte rows, ld = 16, ranks <= 16: eight picks per load instruction and
// half the factor footprint in L2 -- configs 3 and 5, whose factors exceed L2).
template <int P, int NO, bool NAT = false, bool SHORT = false, int LPP = 8>
__global__ void __launch_bounds__(tc_bound_threads(P, NO, NAT, LPP), tc_bound_blocks(P, SHORT, NAT, LPP)) k_update_tc(UpdateArgs a) {
  using W = WarpSmem<1>;  // the per-warp layout does not depend on the rank blocking
  using G = TcGeo<P>;
  constexpr int GP = 8;  // picks per group
  extern __shared__ __align__(16) float smem_f[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int no = NO < NTCB_MAX_ORDER - 1 ? NO : a.no;
  const int R = a.rank;
  const int HS = R | 1;
  const int ld = a.ld;
  float* wbase = smem_f + static_cast<size_t>(wid) * tc_words(no, R, NAT, SHORT);
  float* kt = wbase + tc_ring_words(no, R) + W::batch_words(no);  // NAT: [8][kKtStride]
  uint32_t* st_o = reinterpret_cast<uint32_t*>(wbase);  // [no][kStage]
  float* st_x = wbase + no * W::kStage;                 // [kStage]
  uint32_t* rbat = reinterpret_cast<uint32_t*>(wbase + tc_ring_words(no, R));  // raw batches
  uint32_t* rmsk = rbat + 2 * (no + 1) * 128;                                  // [2][32]
  // the row-end buffers alias the staging ring (drained once an item is streamed)
  float* Hf = wbase;                                                // [R][HS]
  double* gd = reinterpret_cast<double*>(Hf + W::ktile_words(R));  // [64]
  double* vv = gd + 64;                                             // [64]
  const bool full = a.c >= 1.0;
  const int g = lane >> 2;
  const int q0 = 2 * (lane & 3);  // this lane's picks: q0, q0 + 1
  constexpr int NP = P / 2;       // feature-block pairs
  constexpr bool QUAD = P == 4;   // ld == 32: one 128-byte row per pick and mode
  // feature of (lane group gg, block f) -- the rho -> feature map of K'
  auto feat = [&](int gg, int f) {
    return NAT ? gg + 8 * f : QUAD ? 4 * gg + f : (f < 2 * NP ? 16 * (f / 2) + 2 * gg + (f & 1) : 16 * NP + gg);
  };
  int xf = -1;  // block in which this lane holds the x column (feature R)
#pragma unroll
  for (int f = 0; f < P; ++f)
    if (!NAT && feat(g, f) == R) xf = f;
  constexpr int NPS = 32 / LPP;  // NAT: picks per load instruction
  constexpr int NH = 8 / NPS;    // load instructions per group of 8 picks
  const int nq = lane / LPP, nsub = lane % LPP;  // NAT: pick slot (and + NPS), feature quad
  const uint32_t ld4 = static_cast<uint32_t>(ld) * 4u;

  const float* ub2[NO];
  const float* ub1[NO];
#pragma unroll
  for (int m = 0; m < NO; ++m) {
    ub2[m] = a.U[m < no ? m : 0] + (NAT ? 4 * nsub : QUAD ? 4 * g : 2 * g);
    ub1[m] = a.U[m < no ? m : 0] + 16 * NP + g;
  }

  uint64_t stream_policy = 0;
  if constexpr (SHORT) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(stream_policy));
  // Record batches of an item: 128 entries from tb + t into buffer buf
  // (cp.async 16-byte copies of oth[.] and val, the mask word; one group).
  auto fetch_async = [&](uint64_t tb, int hi, int t, int buf) {
    const int r = t + 4 * lane;
    if (r < hi) {
      const uint64_t e = tb + static_cast<uint64_t>(r);
#pragma unroll
      for (int m = 0; m < NO + 1; ++m) {
        if (m < no || m == NO) {
          const int row = (m == NO) ? no : m;
          const void* src = (m == NO) ? static_cast<const void*>(a.val + e) : static_cast<const void*>(a.oth[m] + e);
          const unsigned dst = static_cast<unsigned>(
              __cvta_generic_to_shared(rbat + (buf * (no + 1) + row) * 128 + 4 * lane));
          if constexpr (SHORT) {
            // the view stream is read once: evict-first in L2, so it does not
            // push out the factor rows the gathers reuse (config 5's factors
            // exceed L2 and compete with 20 GB of streamed records per mode)
            asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                         "l"(stream_policy));
          } else {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
          }
        }
      }
      // one mask word per 32 entries: lanes 8i copy word i (the other lanes
      // of the octet would copy the same word -- 8-way shared conflicts)
      if (!full && (lane & 7) == 0) {
        const unsigned dm = static_cast<unsigned>(__cvta_generic_to_shared(rmsk + buf * 32 + (lane >> 3)));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dm), "l"(a.mask + (e >> 5)));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  // Items are prefetched one ahead: the next item's index is claimed while the
  // current one streams, and its first batch is copied in while the current
  // row is finalised (short rows are otherwise a chain of exposed latencies).
  auto claim = [&]() {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(&a.counters[2], 1ull);
    return it;  // lane 0 only; broadcast when needed
  };
  // SHORT (modes of short rows): A and Y of an item's row are copied into
  // pre[parity] with its first batch, for the row-end finalisation
  float* pre = wbase + tc_ring_words(no, R) + W::batch_words(no) + (NAT ? kKtWords : 0);
  int parity = 0;
  auto begin_item = [&](unsigned long long it, WorkItem& w) {
    if (it >= a.n_items) return false;
    w = a.items[it];
    if constexpr (SHORT) {
      if (w.slot < 0 && lane < R) {
        const uint64_t q = w.row * static_cast<uint64_t>(ld) + lane;
        const unsigned dy = static_cast<unsigned>(__cvta_generic_to_shared(pre + parity * 64 + lane));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dy), "l"(a.Y + q));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dy + 128u), "l"(a.A + q));
      }
    }
    const uint64_t tb = w.e0 & ~uint64_t(31);  // 128-byte aligned: one line per quarter-warp cp.async
    fetch_async(tb, static_cast<int>(w.e1 - tb), 0, 0);
    return true;
  };
  WorkItem w;
  bool have = begin_item(__shfl_sync(0xffffffffu, claim(), 0), w);
  while (have) {
    // SHORT: the error key is tested at the end of the item (its load stays
    // off the short item's latency chain)
    unsigned long long err_key = ~0ull;
    if constexpr (SHORT) {
      err_key = *reinterpret_cast<volatile unsigned long long*>(&a.counters[1]);
    } else if (*reinterpret_cast<volatile unsigned long long*>(&a.counters[1]) != ~0ull) {
      asm volatile("cp.async.wait_group 0;\n" ::);
      return;
    }
    const unsigned long long next_it = claim();
    const uint64_t p = w.row;
    const float* my_pre = pre + parity * 64;  // SHORT: this item's A/Y copies
    if constexpr (SHORT) parity ^= 1;

    float acc[G::NT][4];
#pragma unroll
    for (int i = 0; i < G::NT; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][e] = 0.f;

    int head = 0, cnt = 0;  // staging ring [head, head+cnt)

    struct RawPair {
      float f[NO][2][P];  // factor values (mode, pick, feature block)
      float x[2];
    };
    struct RawNat {
      float4 v[NH][NO];  // picks nq (, nq + 4): features 4 nsub .. 4 nsub + 3 of each mode
      float x[NH];
    };
    using Raw = typename std::conditional<NAT, RawNat, RawPair>::type;
    float4 wacc = make_float4(0.f, 0.f, 0.f, 0.f);  // NAT: w = sum x k, features 4 nsub..+3
    auto load_nat = [&](int at, int np) {
      RawNat r;
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int q = nq + NPS * h;
        const bool on = q < np;
        const int sl = (at + q) & (W::kStage - 1);
#pragma unroll
        for (int m = 0; m < NO; ++m)
          if (m < no) {
            const uint32_t row = on ? st_o[m * W::kStage + sl] : 0u;
            r.v[h][m] = __ldg(reinterpret_cast<const float4*>(row_ptr(ub2[m], row, ld4)));
          }
        r.x[h] = on ? st_x[sl] : 0.f;
        if (!on) r.v[h][0] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      return r;
    };
    // gather of one group: np picks present (8 for full groups).  Quad layout
    // (P = 4, ld = 32): one 16-byte load per pick and mode, features 4g..4g+3
    // (a row is one 128-byte line).  Pair layout (P <= 3): block pair
    // (2i, 2i+1) is one 8-byte load (features 16i + 2g, +1), an odd last
    // block one 4-byte load (feature 16 NP + g).  Reads past R hit the row
    // padding or the next row and land in discarded rows/cols of K'^T K'.
    // Group starts are multiples of 8 (head only advances by whole groups
    // inside an item), so the ring pair (q0, q0 + 1) is one 8-byte load.
    auto load_pair = [&](int at, int np) {
      RawPair r;
      const int s0 = (at + q0) & (W::kStage - 1);
      const bool on0 = q0 < np, on1 = q0 + 1 < np;
#pragma unroll
      for (int m = 0; m < NO; ++m)
        if (m < no) {
          const uint2 rr = *reinterpret_cast<const uint2*>(st_o + m * W::kStage + s0);
          const uint32_t rw[2] = {on0 ? rr.x : 0u, on1 ? rr.y : 0u};
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const float* b2 = row_ptr(ub2[m], rw[q], ld4);
            if (QUAD) {
              const float4 v = __ldg(reinterpret_cast<const float4*>(b2));
              r.f[m][q][0] = v.x;
              r.f[m][q][1 % P] = v.y;
              r.f[m][q][2 % P] = v.z;
              r.f[m][q][3 % P] = v.w;
            } else {
#pragma unroll
              for (int i = 0; i < NP; ++i) {
                const float2 v = __ldg(reinterpret_cast<const float2*>(b2) + 8 * i);
                r.f[m][q][2 * i] = v.x;
                r.f[m][q][2 * i + 1] = v.y;
              }
              if (P & 1) r.f[m][q][P - 1] = __ldg(row_ptr(ub1[m], rw[q], ld4));
            }
          }
        }
      const float2 xx = *reinterpret_cast<const float2*>(st_x + s0);
      r.x[0] = on0 ? xx.x : 0.f;
      r.x[1] = on1 ? xx.y : 0.f;
      if (!on0)
#pragma unroll
        for (int f = 0; f < P; ++f) r.f[0][0][f] = 0.f;
      if (!on1)
#pragma unroll
        for (int f = 0; f < P; ++f) r.f[0][1][f] = 0.f;
      return r;
    };
    auto load = [&](int at, int np) {
      if constexpr (NAT)
        return load_nat(at, np);
      else
        return load_pair(at, np);
    };
    // k values of this lane's two picks and feature blocks, fragment layout
    auto kvals = [&](const Raw& r, float (&kf)[2][P]) {
      if constexpr (NAT) {
        // natural layout -> products -> shared tile -> fragment layout
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          float4 k = r.v[h][0];
#pragma unroll
          for (int m = 1; m < NO; ++m)
            if (m < no) {
              k.x *= r.v[h][m].x;
              k.y *= r.v[h][m].y;
              k.z *= r.v[h][m].z;
              k.w *= r.v[h][m].w;
            }
          wacc.x = fmaf(r.x[h], k.x, wacc.x);
          wacc.y = fmaf(r.x[h], k.y, wacc.y);
          wacc.z = fmaf(r.x[h], k.z, wacc.z);
          wacc.w = fmaf(r.x[h], k.w, wacc.w);
          *reinterpret_cast<float4*>(kt + (nq + NPS * h) * kKtStride + 4 * nsub) = k;
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int f = 0; f < P; ++f) kf[q][f] = kt[(q0 + q) * kKtStride + g + 8 * f];
        __syncwarp();  // the tile is rewritten by the next group
      } else {
#pragma unroll
        for (int f = 0; f < P; ++f)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            float k = r.f[0][q][f];
#pragma unroll
            for (int m = 1; m < NO; ++m)
              if (m < no) k *= r.f[m][q][f];
            if (xf == f) k = r.x[q];  // the x column of k'
            kf[q][f] = k;
          }
      }
    };
    auto compute = [&](const Raw& r) {
      uint32_t hb[2][P], hp[P], lp[P];
      float kf[2][P];
      kvals(r, kf);
#pragma unroll
      for (int f = 0; f < P; ++f) {
        float lo[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const float k = kf[q][f];
          hb[q][f] = __float_as_uint(k) & 0xffffe000u;
          lo[q] = k - __uint_as_float(hb[q][f]);
        }
        hp[f] = pack_bf16(__uint_as_float(hb[0][f]), __uint_as_float(hb[1][f]));
        lp[f] = pack_bf16(lo[0], lo[1]);
      }
#pragma unroll
      for (int tl = 0; tl < G::NT; ++tl) {
        const int i = G::mi(tl), j = G::nj(tl);
        const int m0 = 2 * i, m1 = 2 * i + 1;
        const uint32_t a0 = hb[0][m0], a2 = hb[1][m0];
        const uint32_t a1 = m1 < P ? hb[0][m1 < P ? m1 : 0] : 0u;
        const uint32_t a3 = m1 < P ? hb[1][m1 < P ? m1 : 0] : 0u;
        const uint32_t c1 = m1 < P ? hp[m1 < P ? m1 : 0] : 0u;
        const uint32_t c3 = m1 < P ? lp[m1 < P ? m1 : 0] : 0u;
        // The MMA's fp32 accumulation does not round to nearest: accumulating
        // a whole item (thousands of groups) in its C registers leaves a
        // signed error that grows with the number of groups (measured 7e-5
        // relative on config 4's NAT mode updates, whose w is summed on the
        // CUDA cores, and 3.4e-5 on config 3's mode 2, where the bias only
        // partly cancels between H and the x column).  So each group's
        // products are formed from zero and added to the running sums with
        // round-to-nearest FADDs: ~3e-7 everywhere, for +2.4 % on config 2.
        float t4[4];
        mma_tf32_z(t4, a0, a1, a2, a3, hb[0][j], hb[1][j]);
        mma_bf16(t4, hp[m0], c1, lp[m0], c3, lp[j], hp[j]);
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[tl][e] += t4[e];
      }
    };
    // all staged full groups, three-way rotation (two gathers in flight)
    auto drain_full = [&]() {
      const int ng = cnt / GP;
      if (ng == 0) return;
      int al = head;
      Raw r0, r1, r2;
      r0 = load(al, GP);
      al = (al + GP) & (W::kStage - 1);
      if (1 < ng) {
        r1 = load(al, GP);
        al = (al + GP) & (W::kStage - 1);
      }
      for (int gi = 0; gi < ng; gi += 3) {
        if (gi + 2 < ng) {
          r2 = load(al, GP);
          al = (al + GP) & (W::kStage - 1);
        }
        compute(r0);
        if (gi + 1 < ng) {
          if (gi + 3 < ng) {
            r0 = load(al, GP);
            al = (al + GP) & (W::kStage - 1);
          }
          compute(r1);
          if (gi + 2 < ng) {
            if (gi + 4 < ng) {
              r1 = load(al, GP);
              al = (al + GP) & (W::kStage - 1);
            }
            compute(r2);
          }
        }
      }
      head = (head + ng * GP) & (W::kStage - 1);
      cnt -= ng * GP;
    };

    // ---- stream the item in batches of 128 entries (as k_update); batch 0
    // is already in flight (begin_item) ----------------------------------------
    const uint64_t tb = w.e0 & ~uint64_t(31);
    const int lo = static_cast<int>(w.e0 - tb);
    const int hi = static_cast<int>(w.e1 - tb);
    const uint32_t sh0 = static_cast<uint32_t>(tb & 31u);
    int buf = 0;
    for (int t0 = 0; t0 < hi; t0 += 128, buf ^= 1) {
      if (t0 + 128 < hi) {
        fetch_async(tb, hi, t0 + 128, buf ^ 1);
        asm volatile("cp.async.wait_group 1;\n" ::);
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::);
      }
      uint4 co[NO];
#pragma unroll
      for (int m = 0; m < NO; ++m)
        if (m < no) co[m] = reinterpret_cast<const uint4*>(rbat + (buf * (no + 1) + m) * 128)[lane];
      const uint4 cv = reinterpret_cast<const uint4*>(rbat + (buf * (no + 1) + no) * 128)[lane];
      const int r = t0 + 4 * lane;
      uint32_t bits = full ? 0xfu : (rmsk[buf * 32 + (lane >> 3)] >> ((sh0 + static_cast<uint32_t>(r)) & 31u)) & 0xfu;
      if (r < lo) bits &= 0xfu << (lo - r);
      if (r + 4 > hi) bits &= hi - r > 0 ? (0xfu >> (4 - (hi - r))) : 0u;
      cnt += stage_sampled<NO, W::kStage>(bits, co, cv, no, lane, head + cnt, st_o, st_x);
      __syncwarp();
      drain_full();
    }
    if (cnt > 0) {  // the item's last, partial group
      const Raw rp = load(head, cnt);
      compute(rp);
      head = (head + cnt) & (W::kStage - 1);
      cnt = 0;
    }
    // next item: its first batch lands while this row is finalised
    const WorkItem cur = w;
    __syncwarp();
    have = begin_item(__shfl_sync(0xffffffffu, next_it, 0), w);

    // ---- accumulators -> Hf (mirrored upper triangle) and w ----------------
#pragma unroll
    for (int tl = 0; tl < G::NT; ++tl) {
      const int i = G::mi(tl), j = G::nj(tl);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int fb = 2 * i + ((e & 2) ? 1 : 0);  // row block
        const int gc = 2 * (lane & 3) + (e & 1);   // col lane group
        const int rho_r = 8 * fb + g, rho_c = 8 * j + gc;
        if (fb >= P || rho_r > rho_c) continue;  // each unordered pair once
        const int fr = feat(g, fb), fc = feat(gc, j);
        const float v = acc[tl][e];
        if (fr < R && fc < R) {
          Hf[fr * HS + fc] = v;
          Hf[fc * HS + fr] = v;
        } else if (!NAT && fr < R && fc == R) {
          gd[fr] = static_cast<double>(v);
        } else if (!NAT && fc < R && fr == R) {
          gd[fc] = static_cast<double>(v);
        }
      }
    }
    if constexpr (NAT) {
      // w: sum the pick slots holding the same features (lanes nsub + LPP q)
#pragma unroll
      for (int o = LPP; o < 32; o <<= 1) {
        wacc.x += __shfl_xor_sync(0xffffffffu, wacc.x, o);
        wacc.y += __shfl_xor_sync(0xffffffffu, wacc.y, o);
        wacc.z += __shfl_xor_sync(0xffffffffu, wacc.z, o);
        wacc.w += __shfl_xor_sync(0xffffffffu, wacc.w, o);
      }
      if (nq == 0) {
        const float wv[4] = {wacc.x, wacc.y, wacc.z, wacc.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (4 * nsub + i < R) gd[4 * nsub + i] = static_cast<double>(wv[i]);
      }
      wacc = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();
    if (cur.slot < 0) {
      if constexpr (SHORT)
        row_end<true, (P <= 4 ? 8 * P : 0)>(a, p, Hf, gd, vv, lane, my_pre);
      else
        row_end<false, (P <= 4 ? 8 * P : 0)>(a, p, Hf, gd, vv, lane);
    } else {
      float* dst = a.partial + static_cast<uint64_t>(cur.slot) * (R * R + R);
      for (int i = lane; i < R * R; i += 32) dst[i] = Hf[(i / R) * HS + (i % R)];
      for (int r = lane; r < R; r += 32) dst[R * R + r] = static_cast<float>(gd[r]);
    }
    __syncwarp();
    if constexpr (SHORT) {
      if (err_key != ~0ull) {
        asm volatile("cp.async.wait_group 0;\n" ::);
        return;
      }
    }
  }
  peer_fence_at_exit(a);
}

// Rows split across several items: a CTA per row sums its partial slots --
// warp w takes the contiguous slot range w of 8, lanes the elements, every
// load of a slot in flight at once -- then the 8 warp sums are combined in
// warp order in shared memory (deterministic: the association depends only
// on the slot count) and warp 0 runs the same finalisation.
constexpr int kFinPass = 512;  // elements per pass (16 per lane)
// per-warp shared words of the finalise kernels: Hf (R x HS), then gd and vv
// (64 doubles each).  (They used to carry the update kernel's whole per-warp
// layout -- 9 KB at rank 20 -- which kept two thirds of the rows' warps off
// the SMs: the row end is a chain of fp64 latencies, so residency is speed.)
__host__ __device__ constexpr int fin_words(int R) { return WarpSmem<1>::ktile_words(R) + 64 * 2 * 2; }
constexpr int kFinSmall = 16;  // rows with at most this many slots: a warp each
#ifndef NTCB_FINQ
#define NTCB_FINQ 8
#endif
constexpr int kFinQ = NTCB_FINQ;  // slots whose loads are in flight together in k_finalize_small

// 64 registers: 4 CTAs (32 warps) per SM -- the kernel waits on its slot loads (config 2 4.71 -> 4.62 ms)
template <int LD4>
__global__ void __launch_bounds__(kWarps * 32, 4) k_finalize_small(UpdateArgs a) {
  using W = WarpSmem<LD4>;
  extern __shared__ __align__(16) float smem_f[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int R = a.rank;
  const int HS = R | 1;
  float* Hf = smem_f + static_cast<size_t>(wid) * fin_words(R);
  double* gd = reinterpret_cast<double*>(Hf + W::ktile_words(R));
  double* vv = gd + 64;
  const int NE = R * R + R;
  for (uint64_t f = blockIdx.x * kWarps + wid; f < a.n_fins; f += static_cast<uint64_t>(gridDim.x) * kWarps) {
    if (*reinterpret_cast<volatile unsigned long long*>(&a.counters[1]) != ~0ull) return;
    const FinItem fi = a.fins[f];
    const float* base = a.partial + static_cast<uint64_t>(fi.slot0) * NE;
    // slot sums in slot order; the loads of kFinQ slots x 4 elements per lane are in flight together
    // (rows of up to kFinQ slots -- config 2's five -- take one round of loads per 128 elements)
    for (int i0 = 0; i0 < NE; i0 += 128) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int q = 0; q < fi.nslots; q += kFinQ) {
        float v[kFinQ][4];
#pragma unroll
        for (int qq = 0; qq < kFinQ; ++qq)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + 32 * u + lane;
            v[qq][u] = (q + qq < fi.nslots && i < NE) ? base[static_cast<uint64_t>(q + qq) * NE + i] : 0.f;
          }
#pragma unroll
        for (int qq = 0; qq < kFinQ; ++qq)
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[u] += static_cast<double>(v[qq][u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u + lane;
        if (i < R * R)
          Hf[(i / R) * HS + (i % R)] = static_cast<float>(acc[u]);
        else if (i < NE)
          gd[i - R * R] = acc[u];
      }
    }
    __syncwarp();
    row_end<false, (LD4 <= 8 ? 4 * LD4 : 0)>(a, fi.row, Hf, gd, vv, lane);
    __syncwarp();
  }
  peer_fence_at_exit(a);
}


// Big split rows, level 1: a warp per group of <= kSlotGroup consecutive
// slots sums them in slot order (fp64), 4 elements per lane and 4 slots in
// flight; the whole grid works on the groups of every big row at once (one
// CTA per row summing thousands of slots serially took 1.5 ms for a 9M-entry
// row of config 3 and 5.5 ms per mode-2 update of config 5).
__global__ void __launch_bounds__(kWarps * 32) k_slot_groups(UpdateArgs a) {
  const int lane = threadIdx.x & 31;
  const int NE = a.rank * a.rank + a.rank;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kWarps;
  for (uint64_t gi = blockIdx.x * static_cast<uint64_t>(kWarps) + (threadIdx.x >> 5); gi < a.n_groups; gi += nw) {
    const SlotGroup gr = a.groups[gi];
    const float* base = a.partial + static_cast<uint64_t>(gr.slot0) * NE;
    double* out = a.gpart + static_cast<uint64_t>(gr.out) * NE;
    for (int i0 = 0; i0 < NE; i0 += 128) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int q = 0; q < gr.n; q += 4) {
        float v[4][4];
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + 32 * u + lane;
            v[qq][u] = (q + qq < gr.n && i < NE) ? base[static_cast<uint64_t>(q + qq) * NE + i] : 0.f;
          }
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[u] += static_cast<double>(v[qq][u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u + lane;
        if (i < NE) out[i] = acc[u];
      }
    }
  }
}

template <int LD4>
__global__ void __launch_bounds__(kWarps * 32) k_finalize(UpdateArgs a) {
  using W = WarpSmem<LD4>;
  extern __shared__ __align__(16) float smem_f[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int R = a.rank;
  const int HS = R | 1;
  float* Hf = smem_f;  // warp 0's row-end buffers
  double* gd = reinterpret_cast<double*>(Hf + W::ktile_words(R));
  double* vv = gd + 64;
  double* P = reinterpret_cast<double*>(smem_f + fin_words(R));  // [kWarps][kFinPass]
  const int NE = R * R + R;
  __shared__ int stop;
  for (uint64_t f = blockIdx.x; f < a.n_fins; f += gridDim.x) {
    // one read of the error key for the whole CTA: warps that disagreed on it
    // would leave the barriers below with stale partial sums in P[]
    if (threadIdx.x == 0) stop = *reinterpret_cast<volatile unsigned long long*>(&a.counters[1]) != ~0ull;
    __syncthreads();
    if (stop) return;
    const FinItem fi = a.fins[f];
    // the row's slot-group sums (k_slot_groups), contiguous group ranges per
    // warp, combined in warp order below
    const int chunk = (fi.ngroups + kWarps - 1) / kWarps;
    const int qa = wid * chunk, qb = min(fi.ngroups, qa + chunk);
    for (int e0 = 0; e0 < NE; e0 += kFinPass) {
      double acc[kFinPass / 32];
#pragma unroll
      for (int u = 0; u < kFinPass / 32; ++u) acc[u] = 0.0;
      for (int q = qa; q < qb; ++q) {
        const double* src = a.gpart + static_cast<uint64_t>(fi.g0 + q) * NE + e0;
        double v[kFinPass / 32];
#pragma unroll
        for (int u = 0; u < kFinPass / 32; ++u) v[u] = (e0 + 32 * u + lane < NE) ? src[32 * u + lane] : 0.0;
#pragma unroll
        for (int u = 0; u < kFinPass / 32; ++u) acc[u] += v[u];
      }
#pragma unroll
      for (int u = 0; u < kFinPass / 32; ++u) P[wid * kFinPass + 32 * u + lane] = acc[u];
      __syncthreads();
      for (int i = threadIdx.x; i < kFinPass && e0 + i < NE; i += kWarps * 32) {
        double t = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < kWarps; ++w2) t += P[w2 * kFinPass + i];
        const int e = e0 + i;
        if (e < R * R)
          Hf[(e / R) * HS + (e % R)] = static_cast<float>(t);
        else
          gd[e - R * R] = t;
      }
      __syncthreads();
    }
    if (wid == 0) row_end<false, (LD4 <= 8 ? 4 * LD4 : 0)>(a, fi.row, Hf, gd, vv, lane);
    __syncthreads();
  }
  peer_fence_at_exit(a);
}

// ---------------------------------------------------------------------------
// Host side: work lists (cached per mode/row range/c) and launches.
// ---------------------------------------------------------------------------
struct WorkPlan {
  WorkItem* d_items = nullptr;
  FinItem* d_fins = nullptr;  // [n_small small rows][n_fins - n_small big rows]
  SlotGroup* d_groups = nullptr;
  uint64_t n_items = 0, n_fins = 0, n_slots = 0, n_small = 0, n_groups = 0;
  uint64_t n_entries = 0;  // entries over all items
};
using WorkPlans = std::map<std::tuple<const void*, int, uint64_t, uint64_t, uint64_t>, WorkPlan>;

// Segment length of a mode: a function of the WHOLE mode view and the
// device's SM count only -- never of the row range a call covers -- so every
// row is cut into the same items, and its partial sums are associated the same
// way, under any row partition: results are bitwise identical for 1, 2, 4 or
// 8 GPUs (the reference's thread/schedule invariance, nmc.hpp:89-92,
// test_nmc.cpp:337-358).  The length targets ~4 items per resident warp on
// the thinnest shard the box runs (1/8 of the view), at least 2048 entries
// (256 for views under 4M entries, e.g. config 1, whose 2500-entry rows were
// latency bound on one warp) and at most kSeg.
uint64_t segment_length(const ntcb_context* ctx, int mode) {
  const uint64_t* off = ctx->views[mode].h_off;
  const uint64_t total = off[ctx->views[mode].rows] - off[0];
  constexpr uint64_t kMaxShards = 8;
  const uint64_t target = 4ull * static_cast<uint64_t>(ctx->sm_count) * 2 * kWarps * kMaxShards;
  const uint64_t want = (total / target + 127) / 128 * 128;
  return std::min<uint64_t>(kSeg, std::max<uint64_t>(total < (4ull << 20) ? 256 : 2048, want));
}

// Work items of rows [r0, r1): a row of up to segment_length() entries is
// one item, finalised in place; a longer row is cut into items of that
// length from its start (their partial sums go to slots, summed in fp64 by
// the finalise kernels in a fixed order).  The cut depends on the row and
// the mode only, never on [r0, r1): any row partition gives the same bits.
static WorkPlan& plan_for(ntcb_context* ctx, int mode, uint64_t r0, uint64_t r1, double c) {
  uint64_t cbits;
  std::memcpy(&cbits, &c, 8);
  auto& g_plans = ctx_cache<WorkPlans>(ctx, kCacheUpdate);
  auto key = std::make_tuple(static_cast<const void*>(ctx->views[mode].off), mode, r0, r1, cbits);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) return it->second;
  const uint64_t* off = ctx->views[mode].h_off;
  std::vector<WorkItem> items;
  std::vector<FinItem> fins;
  int64_t slot = 0;
  const uint64_t seg = segment_length(ctx, mode);
  for (uint64_t p = r0; p < r1; ++p) {
    const uint64_t n = off[p + 1] - off[p];
    if (blocksize_for(c, n) == 0) continue;  // skipped row (nmc.cpp:237)
    if (n <= seg) {
      items.push_back({p, off[p], off[p + 1], -1});
    } else {
      const uint64_t ns = (n + seg - 1) / seg;
      fins.push_back({p, slot, static_cast<int32_t>(ns), 0, 0});
      for (uint64_t s = 0; s < ns; ++s)
        items.push_back({p, off[p] + s * seg, std::min(off[p + 1], off[p] + (s + 1) * seg), slot++});
    }
  }
  // longest items first: better tail balance for the dynamic scheduler
  if (ctx->tune.item_order == 1) {
    // chunk-major among equal lengths: chunk s of every row is scheduled
    // together, so the warps resident on an SM walk the same window of the
    // slowest-varying other coordinate and its factor rows hit L1 (the order
    // of the items never changes a result: every item owns its slot)
    std::stable_sort(items.begin(), items.end(), [&](const WorkItem& x, const WorkItem& y) {
      const uint64_t lx = x.e1 - x.e0, ly = y.e1 - y.e0;
      if (lx != ly) return lx > ly;
      return (x.e0 - off[x.row]) < (y.e0 - off[y.row]);
    });
  } else {
    std::stable_sort(items.begin(), items.end(), [](const WorkItem& x, const WorkItem& y) {
      return (x.e1 - x.e0) > (y.e1 - y.e0);
    });
  }
  WorkPlan pl;
  pl.n_items = items.size();
  std::stable_partition(fins.begin(), fins.end(), [](const FinItem& f) { return f.nslots <= kFinSmall; });
  pl.n_fins = fins.size();
  pl.n_small = static_cast<uint64_t>(
      std::count_if(fins.begin(), fins.end(), [](const FinItem& f) { return f.nslots <= kFinSmall; }));
  pl.n_slots = static_cast<uint64_t>(slot);
  for (const WorkItem& it : items) pl.n_entries += it.e1 - it.e0;
  std::vector<SlotGroup> groups;
  for (auto& f : fins) {
    if (f.nslots <= kFinSmall) continue;
    f.g0 = static_cast<int64_t>(groups.size());
    f.ngroups = (f.nslots + kSlotGroup - 1) / kSlotGroup;
    for (int32_t g = 0; g < f.ngroups; ++g)
      groups.push_back({f.slot0 + static_cast<int64_t>(g) * kSlotGroup, f.g0 + g,
                        std::min<int32_t>(kSlotGroup, f.nslots - g * kSlotGroup), 0});
  }
  pl.n_groups = groups.size();
  if (pl.n_groups) {
    NTCB_CUDA(cudaMalloc(&pl.d_groups, sizeof(SlotGroup) * pl.n_groups));
    NTCB_CUDA(cudaMemcpy(pl.d_groups, groups.data(), sizeof(SlotGroup) * pl.n_groups, cudaMemcpyHostToDevice));
  }
  if (pl.n_items) {
    NTCB_CUDA(cudaMalloc(&pl.d_items, sizeof(WorkItem) * pl.n_items));
    NTCB_CUDA(cudaMemcpy(pl.d_items, items.data(), sizeof(WorkItem) * pl.n_items, cudaMemcpyHostToDevice));
  }
  if (pl.n_fins) {
    NTCB_CUDA(cudaMalloc(&pl.d_fins, sizeof(FinItem) * pl.n_fins));
    NTCB_CUDA(cudaMemcpy(pl.d_fins, fins.data(), sizeof(FinItem) * pl.n_fins, cudaMemcpyHostToDevice));
  }
  return g_plans.emplace(key, pl).first->second;
}

void drop_plans(ntcb_context* ctx) {
  ++ctx->plan_epoch;  // a captured sweep graph must be rebuilt from an uncaptured sweep
  if (!ctx->cache[kCacheUpdate]) return;
  for (auto& kv : ctx_cache<WorkPlans>(ctx, kCacheUpdate)) {
    if (kv.second.d_items) cudaFree(kv.second.d_items);
    if (kv.second.d_fins) cudaFree(kv.second.d_fins);
    if (kv.second.d_groups) cudaFree(kv.second.d_groups);
  }
  ctx_cache_free<WorkPlans>(ctx, kCacheUpdate);
}

// Average item length of a mode over its whole view below the tuning's
// short_row (cached as a host-only pseudo plan, row range ~0..~0).
static bool mode_short_rows(ntcb_context* ctx, int mode, double c) {
  auto& g_plans = ctx_cache<WorkPlans>(ctx, kCacheUpdate);
  uint64_t cbits;
  std::memcpy(&cbits, &c, 8);
  auto key = std::make_tuple(static_cast<const void*>(ctx->views[mode].off), mode, ~0ull, ~0ull, cbits);
  auto it = g_plans.find(key);
  if (it == g_plans.end()) {
    WorkPlan st;
    const uint64_t* off = ctx->views[mode].h_off;
    const uint64_t seg = segment_length(ctx, mode);
    for (uint64_t p = 0; p < ctx->views[mode].rows; ++p) {
      const uint64_t n = off[p + 1] - off[p];
      if (blocksize_for(c, n) == 0) continue;
      st.n_items += (n + seg - 1) / seg;
      st.n_entries += n;
    }
    it = g_plans.emplace(key, st).first;
  }
  const WorkPlan& st = it->second;
  return st.n_items && st.n_entries < static_cast<uint64_t>(ctx->tune.short_row) * st.n_items;
}

template <int LD4, int NO>
static int launch_items(ntcb_context* ctx, UpdateArgs& a, const WorkPlan& pl, size_t smem) {
  constexpr int T = k_update_threads(LD4);
  smem = smem / kWarps * (T / 32);  // per-warp layout
  NTCB_CUDA(cudaFuncSetAttribute(k_update<LD4, NO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  int per_sm = 0;
  NTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_update<LD4, NO>, T, smem));
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (pl.n_items + T / 32 - 1) / (T / 32);
  grid = std::min<uint64_t>(grid, static_cast<uint64_t>(per_sm) * ctx->sm_count);
  grid = std::max<uint64_t>(grid, 1);
  k_update<LD4, NO><<<static_cast<unsigned>(grid), T, smem, ctx->stream>>>(a);
  NTCB_CUDA(cudaGetLastError());
  return 1;
}

template <int P, int NO, bool NAT = false, bool SHORT = false, int LPP = 8>
static int launch_items_tc(ntcb_context* ctx, UpdateArgs& a, const WorkPlan& pl, size_t smem) {
  // Few items (a small tensor or a thin row shard): fewer warps per CTA so the
  // items spread over every SM instead of filling a few.
  const size_t warp_bytes = smem / kWarps;
  const uint64_t per_sm_items = (pl.n_items + 2 * ctx->sm_count - 1) / (2 * ctx->sm_count);
  // 4-warp CTAs (4 per SM): 3.6 % faster than 8-warp CTAs on config 2 at the
  // same 16 warps/SM (measured); ntcb_tuning.update_wpc overrides for experiments
  const int wmax = ctx->tune.update_wpc;
  const int wpc = static_cast<int>(std::min<uint64_t>(wmax, std::max<uint64_t>(1, per_sm_items)));
  smem = warp_bytes * wpc;
  NTCB_CUDA(cudaFuncSetAttribute(k_update_tc<P, NO, NAT, SHORT, LPP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  NTCB_CUDA(cudaFuncSetAttribute(k_update_tc<P, NO, NAT, SHORT, LPP>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 ctx->tune.update_carveout));
  int per_sm = 0;
  NTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_update_tc<P, NO, NAT, SHORT, LPP>, wpc * 32, smem));
  if (ctx->tune.update_ctas_per_sm > 0) per_sm = std::min(per_sm, ctx->tune.update_ctas_per_sm);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (pl.n_items + wpc - 1) / wpc;
  grid = std::min<uint64_t>(grid, static_cast<uint64_t>(per_sm) * ctx->sm_count);
  grid = std::max<uint64_t>(grid, 1);
  k_update_tc<P, NO, NAT, SHORT, LPP><<<static_cast<unsigned>(grid), wpc * 32, smem, ctx->stream>>>(a);
  NTCB_CUDA(cudaGetLastError());
  return 1;
}

template <int P>
static int launch_tc(ntcb_context* ctx, UpdateArgs& a, const WorkPlan& pl, size_t smem) {
  if (a.no == 1) return launch_items_tc<P, 1>(ctx, a, pl, smem);
  if (a.no == 2) return launch_items_tc<P, 2>(ctx, a, pl, smem);
  return launch_items_tc<P, 3>(ctx, a, pl, smem);
}

// The finalisation launches of a plan: rows split into <= kFinSmall slots (a
// warp each), then slot groups and a CTA per row for the longer ones.
template <int LD4>
static int launch_finalize_ld(ntcb_context* ctx, UpdateArgs& a, const WorkPlan& pl) {
  const size_t smem = static_cast<size_t>(fin_words(a.rank)) * 4 * kWarps;
  int launches = 0;
  if (pl.n_small) {  // warp per row
    NTCB_CUDA(cudaFuncSetAttribute(k_finalize_small<LD4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    UpdateArgs b = a;
    b.fins = pl.d_fins;
    b.n_fins = pl.n_small;
    int per_sm = 0;
    NTCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_finalize_small<LD4>, kWarps * 32, smem));
    const uint64_t fg = std::min<uint64_t>((pl.n_small + kWarps - 1) / kWarps,
                                           static_cast<uint64_t>(ctx->sm_count) * std::max(per_sm, 1));
    k_finalize_small<LD4><<<static_cast<unsigned>(fg), kWarps * 32, smem, ctx->stream>>>(b);
    NTCB_CUDA(cudaGetLastError());
    ++launches;
  }
  if (pl.n_groups) {  // big rows, level 1: slot groups over the whole grid
    const uint64_t gg = std::min<uint64_t>((pl.n_groups + kWarps - 1) / kWarps, static_cast<uint64_t>(ctx->sm_count) * 4);
    k_slot_groups<<<static_cast<unsigned>(gg), kWarps * 32, 0, ctx->stream>>>(a);
    NTCB_CUDA(cudaGetLastError());
    ++launches;
  }
  if (pl.n_fins > pl.n_small) {  // CTA per row
    // warp 0's row-end layout + the per-warp partial sums of one pass
    const size_t fsmem = static_cast<size_t>(fin_words(a.rank)) * 4 + sizeof(double) * kWarps * kFinPass;
    NTCB_CUDA(cudaFuncSetAttribute(k_finalize<LD4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(fsmem)));
    UpdateArgs b = a;
    b.fins = pl.d_fins + pl.n_small;
    b.n_fins = pl.n_fins - pl.n_small;
    const uint64_t fg = std::min<uint64_t>(b.n_fins, static_cast<uint64_t>(ctx->sm_count) * 4);
    k_finalize<LD4><<<static_cast<unsigned>(fg), kWarps * 32, fsmem, ctx->stream>>>(b);
    NTCB_CUDA(cudaGetLastError());
    ++launches;
  }
  return launches;
}

template <int LD4>
static int launch_ld(ntcb_context* ctx, UpdateArgs& a, const WorkPlan& pl) {
  using W = WarpSmem<LD4>;
  const size_t smem = static_cast<size_t>(W::words(a.no, a.rank)) * 4 * kWarps;
  int launches = 0;
  // feature blocks of k' = (k, x), pair layout (the 16-byte quad layout reads
  // whole 128-byte rows and measured 40% slower at rank 20)
  int P = (a.rank + 1 + 7) / 8;
  // tuning knob tc_p = 4 runs the quad layout (one 16-byte load per pick and
  // mode, features 4g..4g+3) at any rank <= 31
  if (ctx->tune.tc_p > P && ctx->tune.tc_p <= 4) P = ctx->tune.tc_p;
  // ranks 32-39 (P = 5) compile but stay on the CUDA-core kernel: at one CTA
  // per SM the pair-layout gathers of three factors measured 21 ms vs 17.6 ms
  // per mode on config 4
  const bool g_tc_off = ctx->tune.no_tc != 0;  // A/B switch: CUDA-core Gram
  const bool nat_off = ctx->tune.no_nat != 0;  // A/B switch
  // modes whose items average fewer than short_row entries over the WHOLE
  // view (a property of the mode, not of a shard: the instantiation must not
  // depend on the partition) -- per-row latencies dominate there
  const bool short_rows = mode_short_rows(ctx, a.mode, a.c);
  if (pl.n_items) prof_kernel_mark(ctx);
  if (pl.n_items && !g_tc_off && !nat_off && a.ld == 16 && ctx->nat_padded && a.rank <= 16 &&
      (a.no == 2 || a.no == 3)) {
    // ranks 9-16 on 64-byte rows: NAT with four lanes per pick
    const bool shrt = short_rows && a.no == 2 && NTCB_NAT4_SHORT;
    const size_t ts = static_cast<size_t>(tc_words(a.no, a.rank, true, shrt)) * 4 * kWarps;
    launches += shrt        ? launch_items_tc<2, 2, true, true, 4>(ctx, a, pl, ts)
                : a.no == 2 ? launch_items_tc<2, 2, true, false, 4>(ctx, a, pl, ts)
                            : launch_items_tc<2, 3, true, false, 4>(ctx, a, pl, ts);
  } else if (pl.n_items && !g_tc_off && !nat_off && a.ld == 32 && (a.rank >= 25 || ctx->nat_padded) &&
      (a.no == 2 || a.no == 3)) {
    // ranks 25-32 (and 9-24 with nat_pad's 128-byte rows): natural-layout
    // gathers through a shared tile into the tensor-core Gram (w on the CUDA
    // cores); P = feature blocks of 8 (no x column)
    const size_t ts = static_cast<size_t>(tc_words(a.no, a.rank, true)) * 4 * kWarps;
    const int pn = (a.rank + 7) / 8;
    if (a.no == 2)
      launches += pn == 2 ? launch_items_tc<2, 2, true>(ctx, a, pl, ts)
                : pn == 3 ? launch_items_tc<3, 2, true>(ctx, a, pl, ts)
                          : launch_items_tc<4, 2, true>(ctx, a, pl, ts);
    else
      launches += pn == 2 ? launch_items_tc<2, 3, true>(ctx, a, pl, ts)
                : pn == 3 ? launch_items_tc<3, 3, true>(ctx, a, pl, ts)
                          : launch_items_tc<4, 3, true>(ctx, a, pl, ts);
  } else if (pl.n_items && short_rows && a.no == 2 && (P == 2 || P == 3) && !g_tc_off) {
    // order 3, ranks 8-23, short rows on average (Zipf tails: configs 3 and
    // 5): the variant that stages each row's A and Y with its first batch
    const size_t ts = static_cast<size_t>(tc_words(a.no, a.rank, false, true)) * 4 * kWarps;
    launches += P == 2 ? launch_items_tc<2, 2, false, true>(ctx, a, pl, ts) : launch_items_tc<3, 2, false, true>(ctx, a, pl, ts);
  } else if (pl.n_items && a.rank <= 31 && a.no <= 3 && !g_tc_off) {  // orders 2 to 4
    const size_t ts = static_cast<size_t>(tc_words(a.no, a.rank)) * 4 * kWarps;
    launches += P == 1 ? launch_tc<1>(ctx, a, pl, ts)
              : P == 2 ? launch_tc<2>(ctx, a, pl, ts)
              : P == 3 ? launch_tc<3>(ctx, a, pl, ts)
                       : launch_tc<4>(ctx, a, pl, ts);
  } else if (pl.n_items) {
    if (a.no == 2)
      launches += launch_items<LD4, 2>(ctx, a, pl, smem);
    else if (a.no == 3)
      launches += launch_items<LD4, 3>(ctx, a, pl, smem);
    else
      launches += launch_items<LD4, NTCB_MAX_ORDER - 1>(ctx, a, pl, smem);
  }
  if (pl.n_items) prof_kernel_mark(ctx);
  launches += launch_finalize_ld<LD4>(ctx, a, pl);
  return launches;
}

static int launch_plan(ntcb_context* ctx, int mode, const WorkPlan& pl, const ntcb_nmc_config& cfg,
                       const uint32_t* mask, float* slots_out);

int launch_update(ntcb_context* ctx, int mode, uint64_t row_begin, uint64_t row_end,
                  const ntcb_nmc_config& cfg, const uint32_t* mask) {
  if (row_end <= row_begin) return 0;
  const WorkPlan& pl = plan_for(ctx, mode, row_begin, row_end, cfg.c);
  if (pl.n_items == 0) return 0;
  return launch_plan(ctx, mode, pl, cfg, mask, nullptr);
}

// Chunks [cb, ce) of one row -- the row's segment_length() pieces from its
// start, exactly the items a whole-row plan cuts it into -- with their fp32
// (H, w) partials written to slots_out[(chunk - cb) (R^2 + R)] and nothing
// finalised: a heavy row shared by several ranks.  The same kernel
// instantiation as the whole-mode plans, so the partials are the bits the
// single-GPU run sums.
int launch_update_chunks(ntcb_context* ctx, int mode, uint64_t row, uint32_t cb, uint32_t ce,
                         const ntcb_nmc_config& cfg, const uint32_t* mask, float* slots_out) {
  const uint64_t* off = ctx->views[mode].h_off;
  const uint64_t seg = segment_length(ctx, mode), n = off[row + 1] - off[row];
  const uint64_t ns = (n + seg - 1) / seg;
  if (ce > ns || cb >= ce) fail(NTCB_ERANGE, "s_nmc_chunks: chunk range out of bounds");
  uint64_t cbits;
  std::memcpy(&cbits, &cfg.c, 8);
  auto& g_plans = ctx_cache<WorkPlans>(ctx, kCacheUpdate);
  auto key = std::make_tuple(static_cast<const void*>(ctx->views[mode].off), mode + 128, row,
                             (static_cast<uint64_t>(cb) << 32) | ce, cbits);
  auto it = g_plans.find(key);
  if (it == g_plans.end()) {
    std::vector<WorkItem> items;
    for (uint64_t s = cb; s < ce; ++s)
      items.push_back({row, off[row] + s * seg, std::min(off[row + 1], off[row] + (s + 1) * seg),
                       static_cast<int64_t>(s - cb)});
    std::stable_sort(items.begin(), items.end(), [](const WorkItem& x, const WorkItem& y) {
      return (x.e1 - x.e0) > (y.e1 - y.e0);
    });
    WorkPlan pl;
    pl.n_items = items.size();
    pl.n_slots = ce - cb;
    for (const WorkItem& w : items) pl.n_entries += w.e1 - w.e0;
    NTCB_CUDA(cudaMalloc(&pl.d_items, sizeof(WorkItem) * pl.n_items));
    NTCB_CUDA(cudaMemcpy(pl.d_items, items.data(), sizeof(WorkItem) * pl.n_items, cudaMemcpyHostToDevice));
    it = g_plans.emplace(key, pl).first;
  }
  return launch_plan(ctx, mode, it->second, cfg, mask, slots_out);
}

// A shared row's complete slot set (its chunks in order, fp32) summed in the
// canonical order -- a warp in slot order up to kFinSmall slots, slot groups
// then group order above, as the whole-mode plans do -- and finalised (power
// method, step, momentum, peer stores).  Y = A (a_init) for the row first.
int launch_finalize_row(ntcb_context* ctx, int mode, uint64_t row, const float* slots, uint32_t nslots,
                        const ntcb_nmc_config& cfg) {
  const uint64_t R = ctx->rank, NE = R * R + R, ld = ctx->ld;
  NTCB_CUDA(cudaMemcpyAsync(ctx->Y[mode] + row * ld, ctx->A[mode] + row * ld, sizeof(float) * ld,
                            cudaMemcpyDeviceToDevice, ctx->stream));
  uint64_t cbits;
  std::memcpy(&cbits, &cfg.c, 8);
  auto& g_plans = ctx_cache<WorkPlans>(ctx, kCacheUpdate);
  auto key = std::make_tuple(static_cast<const void*>(ctx->views[mode].off), mode + 192, row,
                             static_cast<uint64_t>(nslots), cbits);
  auto it = g_plans.find(key);
  if (it == g_plans.end()) {
    WorkPlan pl;
    FinItem f{row, 0, static_cast<int32_t>(nslots), 0, 0};
    std::vector<SlotGroup> groups;
    if (nslots > static_cast<uint32_t>(kFinSmall)) {
      f.ngroups = static_cast<int32_t>((nslots + kSlotGroup - 1) / kSlotGroup);
      for (int32_t g = 0; g < f.ngroups; ++g)
        groups.push_back({static_cast<int64_t>(g) * kSlotGroup, g,
                          std::min<int32_t>(kSlotGroup, static_cast<int32_t>(nslots) - g * kSlotGroup), 0});
    } else {
      pl.n_small = 1;
    }
    pl.n_fins = 1;
    pl.n_groups = groups.size();
    NTCB_CUDA(cudaMalloc(&pl.d_fins, sizeof(FinItem)));
    NTCB_CUDA(cudaMemcpy(pl.d_fins, &f, sizeof(FinItem), cudaMemcpyHostToDevice));
    if (pl.n_groups) {
      NTCB_CUDA(cudaMalloc(&pl.d_groups, sizeof(SlotGroup) * pl.n_groups));
      NTCB_CUDA(cudaMemcpy(pl.d_groups, groups.data(), sizeof(SlotGroup) * pl.n_groups, cudaMemcpyHostToDevice));
    }
    it = g_plans.emplace(key, pl).first;
  }
  const WorkPlan& pl = it->second;
  if (pl.n_groups && ctx->partial_n < 2 * pl.n_groups * NE) {  // fp64 group sums
    if (ctx->partial) cudaFree(ctx->partial);
    NTCB_CUDA(cudaMalloc(&ctx->partial, sizeof(float) * 2 * pl.n_groups * NE));
    ctx->partial_n = 2 * pl.n_groups * NE;
  }
  UpdateArgs a{};
  a.no = ctx->order - 1;
  a.mode = mode;
  a.rank = static_cast<int>(R);
  a.ld = static_cast<int>(ld);
  a.A = ctx->A[mode];
  a.Y = ctx->Y[mode];
  a.n_peers = ctx->n_peers[mode];
  a.peer_fence = ctx->tune.peer_fence;
  for (int q = 0; q < 7; ++q) a.peerA[q] = ctx->peerA[mode][q];
  a.partial = const_cast<float*>(slots);
  a.gpart = reinterpret_cast<double*>(ctx->partial);
  a.groups = pl.d_groups;
  a.n_groups = pl.n_groups;
  a.fins = pl.d_fins;
  a.n_fins = 1;
  a.c = cfg.c;
  a.lambda = cfg.lambda;
  a.power_tol = cfg.power_tol;
  a.power_iters = cfg.power_iters;
  a.counters = ctx->counters;
  const int LD4 = static_cast<int>(ld / 4);
  switch (LD4) {
#define NTCB_LD(x) \
  case x:          \
    return launch_finalize_ld<x>(ctx, a, pl);
    NTCB_LD(1) NTCB_LD(2) NTCB_LD(3) NTCB_LD(4) NTCB_LD(5) NTCB_LD(6) NTCB_LD(7) NTCB_LD(8)
    NTCB_LD(9) NTCB_LD(10) NTCB_LD(11) NTCB_LD(12) NTCB_LD(13) NTCB_LD(14) NTCB_LD(15) NTCB_LD(16)
#undef NTCB_LD
    default:
      fail(NTCB_EINVAL, "s_nmc: rank exceeds the supported maximum (64)");
  }
}

static int launch_plan(ntcb_context* ctx, int mode, const WorkPlan& pl, const ntcb_nmc_config& cfg,
                       const uint32_t* mask, float* slots_out) {
  const DeviceView& v = ctx->views[mode];
  const uint64_t R = ctx->rank;
  if (pl.n_slots && !slots_out) {
    // slots (fp32), then the slot-group sums (fp64) of the big rows
    const uint64_t slot_words = (pl.n_slots * (R * R + R) + 1) & ~1ull;
    const uint64_t need = slot_words + 2 * pl.n_groups * (R * R + R);
    if (ctx->partial_n < need) {
      if (ctx->partial) cudaFree(ctx->partial);
      NTCB_CUDA(cudaMalloc(&ctx->partial, sizeof(float) * need));
      ctx->partial_n = need;
    }
  }
  UpdateArgs a{};
  a.off = v.off;
  a.no = ctx->order - 1;
  int k = 0;
  for (int m = 0; m < ctx->order; ++m)
    if (m != mode) {
      a.oth[k] = v.oth[k];
      a.U[k] = ctx->A[m];
      ++k;
    }
  a.val = v.val;
  a.mask = mask;
  a.mode = mode;
  a.rank = static_cast<int>(R);
  a.ld = static_cast<int>(ctx->ld);
  a.A = ctx->A[mode];
  a.Y = ctx->Y[mode];
  a.n_peers = ctx->n_peers[mode];
  a.peer_fence = ctx->tune.peer_fence;
  for (int q = 0; q < 7; ++q) a.peerA[q] = ctx->peerA[mode][q];
  a.items = pl.d_items;
  a.n_items = pl.n_items;
  a.fins = pl.d_fins;
  a.n_fins = pl.n_fins;
  a.partial = slots_out ? slots_out : ctx->partial;
  a.gpart = pl.n_groups ? reinterpret_cast<double*>(ctx->partial + ((pl.n_slots * (R * R + R) + 1) & ~1ull)) : nullptr;
  a.groups = pl.d_groups;
  a.n_groups = pl.n_groups;
  a.c = cfg.c;
  a.lambda = cfg.lambda;
  a.power_tol = cfg.power_tol;
  a.power_iters = cfg.power_iters;
  a.counters = ctx->counters;
  // reset the work cursor
  NTCB_CUDA(cudaMemsetAsync(ctx->counters + 2, 0, sizeof(unsigned long long), ctx->stream));
  const int LD4 = static_cast<int>(ctx->ld / 4);
  switch (LD4) {
#define NTCB_LD(x) \
  case x:          \
    return launch_ld<x>(ctx, a, pl);
    NTCB_LD(1) NTCB_LD(2) NTCB_LD(3) NTCB_LD(4) NTCB_LD(5) NTCB_LD(6) NTCB_LD(7) NTCB_LD(8)
    NTCB_LD(9) NTCB_LD(10) NTCB_LD(11) NTCB_LD(12) NTCB_LD(13) NTCB_LD(14) NTCB_LD(15) NTCB_LD(16)
#undef NTCB_LD
    default:
      fail(NTCB_EINVAL, "s_nmc: rank exceeds the supported maximum (64)");
  }
}

}  // namespace ntcb
