// Device construction of the canonical tensor and its mode views.
//
// Replaces, on the device, ntc::SparseTensor's constructor
// (sparse_tensor.cpp:24-73: validation, lexicographic sort, duplicate
// rejection) and build_mode_views (mode_view.cpp:8-37: stable counting sort
// by the mode coordinate).  Because keys are unique, view m is exactly the
// entry list sorted by (i_m, remaining coordinates in ascending mode order),
// i.e. a STABLE sort of the lexicographic order by i_m -- done here as LSD
// radix passes (CUB onesweep, the CUDA toolkit's device radix sort) over
// packed coordinate keys.  The resulting permutation is bit-identical to the
// reference's (tests/test_gpu_parity.py::test_views_bit_exact).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"

namespace ntcb {

namespace {

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  explicit DevBuf(size_t count) : n(count) {
    if (count) NTCB_CUDA(cudaMalloc(&p, sizeof(T) * count));
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

int bits_for(uint64_t d) {  // bits needed for coordinates 0..d-1
  int b = 1;
  while (b < 64 && (d - 1) >> b) ++b;
  return b;
}

// first invalid entry: key = e*4 + kind  (kind 0 bounds, 1 non-finite, 2 negative)
template <class VT>
__global__ void k_validate(const uint32_t* idx, const VT* vals, uint64_t nnz, int order,
                           const uint64_t* dims, unsigned long long* first_bad) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    int kind = -1;
    for (int m = 0; m < order; ++m)
      if (idx[e * order + m] >= dims[m]) {
        kind = 0;
        break;
      }
    if (kind < 0) {
      const double v = static_cast<double>(vals[e]);
      if (!isfinite(v))
        kind = 1;
      else if (v < 0.0)
        kind = 2;
    }
    if (kind >= 0) atomicMin(first_bad, static_cast<unsigned long long>(e) * 4 + kind);
  }
}

__global__ void k_to_f32(const double* in, float* out, uint64_t n) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[e] = static_cast<float>(in[e]);
}

__global__ void k_iota(uint32_t* p, uint64_t n) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[e] = static_cast<uint32_t>(e);
}

// key[e] = packed coordinates modes [m0, m1) of entry perm[e]
__global__ void k_pack_keys(const uint32_t* idx, const uint32_t* perm, uint64_t nnz, int order,
                            int m0, int m1, const int* shift, uint64_t* key) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t* ix = idx + static_cast<uint64_t>(perm[e]) * order;
    uint64_t k = 0;
    for (int m = m0; m < m1; ++m) k |= static_cast<uint64_t>(ix[m]) << shift[m];
    key[e] = k;
  }
}

__global__ void k_mode_keys(const uint32_t* idx, const uint32_t* perm, uint64_t nnz, int order,
                            int mode, uint32_t* key) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    key[e] = idx[static_cast<uint64_t>(perm[e]) * order + mode];
}

// first duplicate in lexicographic order (position of the later copy)
__global__ void k_dups(const uint32_t* idx, const uint32_t* perm, uint64_t nnz, int order,
                       unsigned long long* first_dup) {
  for (uint64_t e = 1 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t* a = idx + static_cast<uint64_t>(perm[e - 1]) * order;
    const uint32_t* b = idx + static_cast<uint64_t>(perm[e]) * order;
    bool eq = true;
    for (int m = 0; m < order; ++m) eq &= (a[m] == b[m]);
    if (eq) atomicMin(first_dup, static_cast<unsigned long long>(e));
  }
}

// offsets[p] = first position whose sorted key >= p (p in [0, rows])
__global__ void k_offsets(const uint32_t* skey, uint64_t nnz, uint64_t rows, uint64_t* off) {
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p <= rows;
       p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (skey[mid] < p)
        lo = mid + 1;
      else
        hi = mid;
    }
    off[p] = lo;
  }
}

// SoA view records: oth[k][t], val[t] for entry perm[t]
__global__ void k_gather_view(const uint32_t* idx, const float* vals, const uint32_t* perm,
                              uint64_t nnz, int order, int mode, uint32_t** oth, float* val) {
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < nnz;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t e = perm[t];
    const uint32_t* ix = idx + e * order;
    int k = 0;
    for (int m = 0; m < order; ++m)
      if (m != mode) oth[k++][t] = ix[m];
    val[t] = vals[e];
  }
}

unsigned grid_for(uint64_t n, int sms) {
  uint64_t g = (n + 255) / 256;
  const uint64_t cap = static_cast<uint64_t>(sms) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

// Stable LSD radix sort of (keys, values) pairs; results land back in the
// input buffers.
template <class KT>
void radix_pairs(ntcb_context* ctx, KT* keys, KT* keys_alt, uint32_t* vals, uint32_t* vals_alt,
                 uint64_t n, int end_bit) {
  cub::DoubleBuffer<KT> dk(keys, keys_alt);
  cub::DoubleBuffer<uint32_t> dv(vals, vals_alt);
  size_t tmp = 0;
  NTCB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, static_cast<int64_t>(n), 0,
                                            end_bit, ctx->stream));
  DevBuf<unsigned char> t(tmp);
  NTCB_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, dk, dv, static_cast<int64_t>(n), 0, end_bit,
                                            ctx->stream));
  if (dk.Current() != keys)
    NTCB_CUDA(cudaMemcpyAsync(keys, dk.Current(), sizeof(KT) * n, cudaMemcpyDeviceToDevice,
                              ctx->stream));
  if (dv.Current() != vals)
    NTCB_CUDA(cudaMemcpyAsync(vals, dv.Current(), sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice,
                              ctx->stream));
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace

void drop_plans(ntcb_context* ctx);
void drop_heavy(ntcb_context* ctx);
void drop_sample_plans(ntcb_context* ctx);
void drop_metric_plans(ntcb_context* ctx);

void free_views(ntcb_context* ctx) {
  drop_plans(ctx);
  drop_heavy(ctx);
  drop_sample_plans(ctx);
  drop_metric_plans(ctx);
  for (int m = 0; m < NTCB_MAX_ORDER; ++m) {
    DeviceView& v = ctx->views[m];
    if (v.off) cudaFree(v.off);
    for (auto& o : v.oth)
      if (o) cudaFree(o + v.a_lo);
    if (v.val) cudaFree(v.val + v.a_lo);
    for (auto& b : ctx->mask[m]) {
      if (b) cudaFree(b + (v.a_lo >> 5));
      b = nullptr;
    }
    delete[] v.h_off;
    v = DeviceView{};
  }
  ctx->mask_words = 0;
  if (ctx->partial) cudaFree(ctx->partial);
  ctx->partial = nullptr;
  ctx->partial_n = 0;
  if (ctx->perm_scratch) cudaFree(ctx->perm_scratch);
  ctx->perm_scratch = nullptr;
  if (ctx->heavy_flags) cudaFree(ctx->heavy_flags);
  ctx->heavy_flags = nullptr;
  ctx->heavy_flags_n = 0;
  ctx->perm_scratch_n = 0;
  ctx->nnz = 0;
  ctx->order = 0;
}

// Builds everything from device COO (idx entry-major u32, vals f32 already
// validated).  Takes ownership of nothing; idx/vals are only read.
void build_views(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                 const uint32_t* d_idx, const float* d_vals) {
  const int sms = ctx->sm_count;
  cudaStream_t st = ctx->stream;
  if (nnz >= (1ull << 32))
    fail(NTCB_EINVAL, "SparseTensor: more than 2^32-1 entries per device is not supported");

  // ---- canonical lexicographic order: LSD passes over packed key groups ----
  DevBuf<uint32_t> perm(nnz), perm_alt(nnz);
  DevBuf<uint64_t> key(nnz), key_alt(nnz);
  if (nnz) {
    k_iota<<<grid_for(nnz, sms), 256, 0, st>>>(perm.p, nnz);
    NTCB_CUDA(cudaGetLastError());
    std::vector<int> bits(order), shift(order, 0);
    for (int m = 0; m < order; ++m) bits[m] = bits_for(dims[m]);
    DevBuf<int> d_shift(order);
    DevBuf<uint64_t> d_dims(order);
    NTCB_CUDA(cudaMemcpyAsync(d_dims.p, dims, sizeof(uint64_t) * order, cudaMemcpyHostToDevice, st));
    // groups from the least significant (last) mode upwards, <= 64 bits each
    int m1 = order;
    while (m1 > 0) {
      int m0 = m1, used = 0;
      while (m0 > 0 && used + bits[m0 - 1] <= 64) {
        used += bits[m0 - 1];
        --m0;
      }
      int s = 0;
      for (int m = m1 - 1; m >= m0; --m) {
        shift[m] = s;
        s += bits[m];
      }
      NTCB_CUDA(cudaMemcpyAsync(d_shift.p, shift.data(), sizeof(int) * order,
                                cudaMemcpyHostToDevice, st));
      k_pack_keys<<<grid_for(nnz, sms), 256, 0, st>>>(d_idx, perm.p, nnz, order, m0, m1,
                                                      d_shift.p, key.p);
      NTCB_CUDA(cudaGetLastError());
      radix_pairs<uint64_t>(ctx, key.p, key_alt.p, perm.p, perm_alt.p, nnz, used);
      m1 = m0;
    }
    // duplicate rejection (sparse_tensor.cpp:67-72)
    unsigned long long* d_dup = reinterpret_cast<unsigned long long*>(key_alt.p);
    NTCB_CUDA(cudaMemsetAsync(d_dup, 0xff, sizeof(unsigned long long), st));
    k_dups<<<grid_for(nnz, sms), 256, 0, st>>>(d_idx, perm.p, nnz, order, d_dup);
    NTCB_CUDA(cudaGetLastError());
    unsigned long long dup = 0;
    NTCB_CUDA(cudaMemcpyAsync(&dup, d_dup, sizeof dup, cudaMemcpyDeviceToHost, st));
    NTCB_CUDA(cudaStreamSynchronize(st));
    if (dup != ~0ull) {
      uint32_t pe = 0;
      NTCB_CUDA(cudaMemcpy(&pe, perm.p + dup, sizeof pe, cudaMemcpyDeviceToHost));
      std::vector<uint32_t> ix(order);
      NTCB_CUDA(cudaMemcpy(ix.data(), d_idx + static_cast<uint64_t>(pe) * order,
                           sizeof(uint32_t) * order, cudaMemcpyDeviceToHost));
      std::string s = "SparseTensor: duplicate index (";
      for (int m = 0; m < order; ++m) s += (m ? "," : "") + std::to_string(ix[m] + 1ull);
      fail(NTCB_EINVAL, s + ")");
    }
  }

  free_views(ctx);
  ctx->order = order;
  ctx->nnz = nnz;
  for (int m = 0; m < order; ++m) ctx->dims[m] = dims[m];

  // ---- per-mode stable views -------------------------------------------------
  // (the lexicographic pass's alternate buffer is free now: it is the mode
  // sorts' alternate, so a 1.7B-entry tensor builds within one device)
  DevBuf<uint32_t> mperm(nnz);
  uint32_t* mperm_alt = perm_alt.p;
  uint32_t* mkey = reinterpret_cast<uint32_t*>(key.p);      // reuse as u32 buffers
  uint32_t* mkey_alt = reinterpret_cast<uint32_t*>(key_alt.p);
  DevBuf<uint32_t*> d_oth(NTCB_MAX_ORDER);
  for (int m = 0; m < order; ++m) {
    DeviceView& v = ctx->views[m];
    v.rows = dims[m];
    v.row_lo = 0;
    v.row_hi = dims[m];
    v.a_lo = 0;
    NTCB_CUDA(cudaMalloc(&v.off, sizeof(uint64_t) * (v.rows + 1)));
    for (int k = 0; k < order - 1; ++k) NTCB_CUDA(cudaMalloc(&v.oth[k], sizeof(uint32_t) * (nnz + kViewPad)));
    NTCB_CUDA(cudaMalloc(&v.val, sizeof(float) * (nnz + kViewPad)));
    if (nnz) {
      NTCB_CUDA(cudaMemcpyAsync(mperm.p, perm.p, sizeof(uint32_t) * nnz, cudaMemcpyDeviceToDevice, st));
      k_mode_keys<<<grid_for(nnz, sms), 256, 0, st>>>(d_idx, mperm.p, nnz, order, m, mkey);
      NTCB_CUDA(cudaGetLastError());
      if (m != 0) radix_pairs<uint32_t>(ctx, mkey, mkey_alt, mperm.p, mperm_alt, nnz, bits_for(dims[m]));
      k_offsets<<<grid_for(v.rows + 1, sms), 256, 0, st>>>(mkey, nnz, v.rows, v.off);
      NTCB_CUDA(cudaGetLastError());
      NTCB_CUDA(cudaMemcpyAsync(d_oth.p, v.oth, sizeof(uint32_t*) * NTCB_MAX_ORDER,
                                cudaMemcpyHostToDevice, st));
      k_gather_view<<<grid_for(nnz, sms), 256, 0, st>>>(d_idx, d_vals, mperm.p, nnz, order, m,
                                                        d_oth.p, v.val);
      NTCB_CUDA(cudaGetLastError());
    } else {
      NTCB_CUDA(cudaMemsetAsync(v.off, 0, sizeof(uint64_t) * (v.rows + 1), st));
    }
    v.h_off = new uint64_t[v.rows + 1];
    NTCB_CUDA(cudaMemcpyAsync(v.h_off, v.off, sizeof(uint64_t) * (v.rows + 1),
                              cudaMemcpyDeviceToHost, st));
    NTCB_CUDA(cudaStreamSynchronize(st));
    uint64_t mx = 0;
    for (uint64_t p = 0; p < v.rows; ++p) mx = std::max(mx, v.h_off[p + 1] - v.h_off[p]);
    v.max_slice = mx;
  }
  ctx->mask_words = nnz / 32 + 2;
  for (int m = 0; m < order; ++m)
    for (int q = 0; q < 2; ++q) {
      NTCB_CUDA(cudaMalloc(&ctx->mask[m][q], sizeof(uint32_t) * ctx->mask_words));
      NTCB_CUDA(cudaMemsetAsync(ctx->mask[m][q], 0, sizeof(uint32_t) * ctx->mask_words, st));
      ctx->consumed_valid[m][q] = false;
    }
  // Per-entry Fisher-Yates scratch for slices beyond the sampler's smem budget.
  uint64_t big = 0;
  for (int m = 0; m < order; ++m) big = std::max(big, ctx->views[m].max_slice);
  if (big > 2048) {
    ctx->perm_scratch_n = nnz;
    NTCB_CUDA(cudaMalloc(&ctx->perm_scratch, sizeof(uint32_t) * std::max<uint64_t>(nnz, 1)));
  }
  NTCB_CUDA(cudaStreamSynchronize(st));
}

// Validates device COO (values of type VT) and converts them to fp32.
template <class VT>
void validate_device(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                     const uint32_t* d_idx, const VT* d_vals) {
  if (order < 2) fail(NTCB_EINVAL, "SparseTensor: order must be >= 2");
  if (order > NTCB_MAX_ORDER) fail(NTCB_EINVAL, "SparseTensor: order exceeds the supported maximum (8)");
  for (int m = 0; m < order; ++m)
    if (dims[m] == 0) fail(NTCB_EINVAL, "SparseTensor: dimensions must be positive");
  for (int m = 0; m < order; ++m)
    if (dims[m] > (1ull << 32)) fail(NTCB_EINVAL, "SparseTensor: dimension exceeds coord_t range");
  if (!nnz) return;
  cudaStream_t st = ctx->stream;
  DevBuf<uint64_t> d_dims(order);
  DevBuf<unsigned long long> d_bad(1);
  NTCB_CUDA(cudaMemcpyAsync(d_dims.p, dims, sizeof(uint64_t) * order, cudaMemcpyHostToDevice, st));
  NTCB_CUDA(cudaMemsetAsync(d_bad.p, 0xff, sizeof(unsigned long long), st));
  k_validate<VT><<<grid_for(nnz, ctx->sm_count), 256, 0, st>>>(d_idx, d_vals, nnz, order,
                                                               d_dims.p, d_bad.p);
  NTCB_CUDA(cudaGetLastError());
  unsigned long long bad = 0;
  NTCB_CUDA(cudaMemcpyAsync(&bad, d_bad.p, sizeof bad, cudaMemcpyDeviceToHost, st));
  NTCB_CUDA(cudaStreamSynchronize(st));
  if (bad != ~0ull) {
    const uint64_t e = bad / 4;
    const int kind = static_cast<int>(bad % 4);
    const char* what = kind == 0 ? "SparseTensor: index out of bounds at entry "
                       : kind == 1 ? "SparseTensor: non-finite value at entry "
                                   : "SparseTensor: negative value at entry ";
    fail(NTCB_EINVAL, what + std::to_string(e));
  }
}

void load_tensor_f64(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                     const uint32_t* h_idx, const double* h_vals) {
  if (order >= 2 && order <= NTCB_MAX_ORDER && nnz) {
    DevBuf<uint32_t> idx(nnz * order);
    DevBuf<double> v64(nnz);
    DevBuf<float> v32(nnz);
    NTCB_CUDA(cudaMemcpyAsync(idx.p, h_idx, sizeof(uint32_t) * nnz * order, cudaMemcpyHostToDevice, ctx->stream));
    NTCB_CUDA(cudaMemcpyAsync(v64.p, h_vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx->stream));
    validate_device<double>(ctx, order, dims, nnz, idx.p, v64.p);
    k_to_f32<<<grid_for(nnz, ctx->sm_count), 256, 0, ctx->stream>>>(v64.p, v32.p, nnz);
    NTCB_CUDA(cudaGetLastError());
    build_views(ctx, order, dims, nnz, idx.p, v32.p);
  } else {
    validate_device<double>(ctx, order, dims, nnz, nullptr, nullptr);
    build_views(ctx, order, dims, nnz, nullptr, nullptr);
  }
}

void load_tensor_f32(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                     const uint32_t* idx, const float* vals, bool on_device) {
  if (order >= 2 && order <= NTCB_MAX_ORDER && nnz) {
    if (on_device) {
      validate_device<float>(ctx, order, dims, nnz, idx, vals);
      build_views(ctx, order, dims, nnz, idx, vals);
      return;
    }
    DevBuf<uint32_t> d_idx(nnz * order);
    DevBuf<float> d_v(nnz);
    NTCB_CUDA(cudaMemcpyAsync(d_idx.p, idx, sizeof(uint32_t) * nnz * order, cudaMemcpyHostToDevice, ctx->stream));
    NTCB_CUDA(cudaMemcpyAsync(d_v.p, vals, sizeof(float) * nnz, cudaMemcpyHostToDevice, ctx->stream));
    validate_device<float>(ctx, order, dims, nnz, d_idx.p, d_v.p);
    build_views(ctx, order, dims, nnz, d_idx.p, d_v.p);
  } else {
    validate_device<float>(ctx, order, dims, nnz, nullptr, nullptr);
    build_views(ctx, order, dims, nnz, nullptr, nullptr);
  }
}

}  // namespace ntcb
