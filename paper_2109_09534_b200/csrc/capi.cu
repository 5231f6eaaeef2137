// C-ABI of ntc-b200 (include/ntc_b200.h): context, tensor/factor residency,
// the S_NMC call sequence, the AO driver and metrics.  Host orchestration
// only; all arithmetic of the path runs in the kernels of sampler.cu,
// update.cu, metrics.cu and tensor.cu.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace ntcb {
int launch_sample(ntcb_context* ctx, cudaStream_t stream, uint32_t* mask, int mode,
                  uint64_t row_begin, uint64_t row_end, double c, uint64_t root,
                  uint32_t* dbg_picks, const uint64_t* dbg_off, int direct = 0);
int launch_update(ntcb_context* ctx, int mode, uint64_t row_begin, uint64_t row_end,
                  const ntcb_nmc_config& cfg, const uint32_t* mask);
int launch_update_chunks(ntcb_context* ctx, int mode, uint64_t row, uint32_t cb, uint32_t ce,
                         const ntcb_nmc_config& cfg, const uint32_t* mask, float* slots_out);
int launch_finalize_row(ntcb_context* ctx, int mode, uint64_t row, const float* slots, uint32_t nslots,
                        const ntcb_nmc_config& cfg);
uint64_t segment_length(const ntcb_context* ctx, int mode);
int launch_sample_set(ntcb_context* ctx, cudaStream_t stream, uint32_t* mask, int mode,
                      uint64_t row_begin, uint64_t row_end, double c, uint64_t root, int direct,
                      uint64_t* heavy_cap);
int launch_sample_heavy(ntcb_context* ctx, cudaStream_t stream, uint32_t* mask, int mode,
                        uint64_t row_begin, uint64_t row_end, double c, uint64_t root, int direct,
                        uint64_t cap);
void free_views(ntcb_context* ctx);
void drop_plans(ntcb_context* ctx);
void drop_heavy(ntcb_context* ctx);
void drop_sample_plans(ntcb_context* ctx);
void drop_metric_plans(ntcb_context* ctx);
void load_tensor_f64(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                     const uint32_t* h_idx, const double* h_vals);
void load_tensor_f32(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                     const uint32_t* idx, const float* vals, bool on_device);
void device_metrics(ntcb_context* ctx, double* sse, double* sumsq, double* reg);
void render_model(ntcb_context* ctx, uint8_t* d_pixels);
void synth_uniform(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                   uint64_t true_rank, double sigma, uint64_t seed);
void synth_general(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                   uint64_t true_rank, double sigma, uint64_t seed, const double* zipf_alpha,
                   int kind);
}  // namespace ntcb

using namespace ntcb;

namespace {

thread_local std::string g_err;

// Per-context host bookkeeping (owned by the context: ctx->host).
struct HostState {
  uint64_t pending_accessed = 0;
  bool verified[NTCB_MAX_ORDER] = {};  // factor rows known nonnegative
  std::map<std::tuple<int, uint64_t, uint64_t, uint64_t>, uint64_t> bs_cache;
  float* stage = nullptr;  // pinned fp32 staging for host-buffer factor transfers
  uint64_t stage_n = 0;    // floats
  cudaGraphExec_t sweep_exec = nullptr;  // the sweep graph (ntcb_tuning.graph)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  uint64_t sweep_warm = 0;  // plan epoch + 1 of the last uncaptured sweep (plans and buffers exist)
  void* io_in = nullptr;   // device fp64 a_init / fp32 scratch / fp64 outputs (pinned-buffer path)
  void* io_f = nullptr;
  void* io_out = nullptr;
  uint64_t io_in_cap = 0, io_f_cap = 0, io_out_cap = 0;  // bytes
  bool queued = false;     // work enqueued since the last collect
  // ntcb_sample_prefetch: the whole-mode sampled set of inner iteration 0 drawn ahead
  struct Prefetch {
    bool valid = false;
    uint64_t rng_state = 0;
    double c = 0.0;
    int parity = 0;
  } prefetch[NTCB_MAX_ORDER];
};
HostState& host_of(ntcb_context* ctx) { return *static_cast<HostState*>(ctx->host); }
// prefetched sampled sets die with the masks / views / plans they were drawn for
void drop_prefetch(ntcb_context* ctx) {
  if (ctx->host)
    for (auto& p : host_of(ctx).prefetch) p.valid = false;
}

#define API_TRY try {
#define API_CATCH                                   \
  }                                                 \
  catch (const ntcb::Error& e) {                    \
    g_err = e.what();                               \
    return e.code;                                  \
  }                                                 \
  catch (const std::exception& e) {                 \
    g_err = e.what();                               \
    return NTCB_ECUDA;                              \
  }                                                 \
  return NTCB_OK;

void need_ctx(ntcb_context* ctx) {
  if (!ctx) fail(NTCB_EINVAL, "ntcb: null context");
  NTCB_CUDA(cudaSetDevice(ctx->device));
}
void need_tensor(ntcb_context* ctx) {
  if (ctx->order < 2) fail(NTCB_EINVAL, "ntcb: no tensor loaded");
}
// rows [r0, r1) of view `mode` must be resident (ntcb_view_keep_rows)
void need_rows(ntcb_context* ctx, int mode, uint64_t r0, uint64_t r1) {
  const DeviceView& v = ctx->views[mode];
  if (r1 > r0 && (r0 < v.row_lo || r1 > v.row_hi))
    fail(NTCB_ERANGE, "ntcb: rows [" + std::to_string(r0) + ", " + std::to_string(r1) + ") of mode " +
                          std::to_string(mode + 1) + " are not resident (slab [" + std::to_string(v.row_lo) +
                          ", " + std::to_string(v.row_hi) + "))");
}
bool is_slab(const ntcb_context* ctx) {
  for (int m = 0; m < ctx->order; ++m)
    if (ctx->views[m].row_lo != 0 || ctx->views[m].row_hi != ctx->views[m].rows) return true;
  return false;
}
void need_whole(ntcb_context* ctx) {
  for (int m = 0; m < ctx->order; ++m) need_rows(ctx, m, 0, ctx->dims[m]);
}

void need_factors(ntcb_context* ctx) {
  need_tensor(ctx);
  if (ctx->rank == 0 || !ctx->A[0]) fail(NTCB_EINVAL, "ntcb: no factors loaded");
}

void validate_nmc(const ntcb_nmc_config* c) {  // NmcConfig::validate, nmc.cpp:13-23
  if (!c) fail(NTCB_EINVAL, "NmcConfig: null");
  if (!(c->lambda > 0.0)) fail(NTCB_EINVAL, "NmcConfig: lambda must be > 0");
  if (!(c->c > 0.0 && c->c <= 1.0)) fail(NTCB_EINVAL, "NmcConfig: c must be in (0, 1]");
  if (c->max_inner < 0) fail(NTCB_EINVAL, "NmcConfig: max_inner must be >= 0");
  if (c->power_iters < 1) fail(NTCB_EINVAL, "NmcConfig: power_iters must be >= 1");
  if (!(c->power_tol > 0.0)) fail(NTCB_EINVAL, "NmcConfig: power_tol must be > 0");
  if (c->threads < 1) fail(NTCB_EINVAL, "NmcConfig: threads must be >= 1");
  if (c->chunk < 0) fail(NTCB_EINVAL, "NmcConfig: chunk must be >= 0");
}

// sum over rows of floor(c * n_p) (nmc.cpp:36-40) -- known before the run.
uint64_t blocksize_sum(ntcb_context* ctx, int mode, uint64_t r0, uint64_t r1, double c) {
  auto& hs = host_of(ctx);
  uint64_t cbits;
  std::memcpy(&cbits, &c, 8);
  auto key = std::make_tuple(mode, r0, r1, cbits);
  auto it = hs.bs_cache.find(key);
  if (it != hs.bs_cache.end()) return it->second;
  const uint64_t* off = ctx->views[mode].h_off;
  uint64_t s = 0;
  for (uint64_t p = r0; p < r1; ++p) s += blocksize_for(c, off[p + 1] - off[p]);
  hs.bs_cache[key] = s;
  return s;
}

void prof_mark(ntcb_context* ctx, int kind, cudaStream_t st) {
  Profile& pf = ctx->prof;
  if (!pf.on) return;
  if (pf.n + 2 > 4096) return;
  NTCB_CUDA(cudaEventRecord(pf.ev[pf.n], st));
  pf.kind[pf.n / 2] = kind;
  pf.n += 1;
}
void prof_end(ntcb_context* ctx, cudaStream_t st) {
  Profile& pf = ctx->prof;
  if (!pf.on || (pf.n & 1) == 0) return;
  NTCB_CUDA(cudaEventRecord(pf.ev[pf.n], st));
  pf.n += 1;
}

// Queue one s_nmc on rows [r0, r1) of `mode` with a_init == factors[mode].
// Sampling runs on the side stream (it never reads factors), so the sample of
// the next mode overlaps this mode's update; events order mask reuse.
// Sampled set of inner iteration `l` into the next mask of `mode` (side
// stream); returns the parity used.  The main stream waits on it later.
int enqueue_sample(ntcb_context* ctx, int mode, uint64_t r0, uint64_t r1, const ntcb_nmc_config& cfg,
                   uint64_t rng_state, int l) {
  const int par = ctx->mask_parity[mode];
  ctx->mask_parity[mode] ^= 1;
  host_of(ctx).prefetch[mode].valid = false;  // its buffer is the next one to be overwritten
  const DeviceView& v = ctx->views[mode];
  const uint64_t e0 = v.h_off[r0], e1 = v.h_off[r1];
  if (cfg.c < 1.0 && e1 > e0) {
    uint32_t* mask = ctx->mask[mode][par];
    const uint64_t root = fork64(rng_state, static_cast<uint64_t>(l));
    if (ctx->consumed_valid[mode][par])
      NTCB_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_consumed[mode][par], 0));
    const uint64_t w0 = e0 >> 5, w1 = ((e1 - 1) >> 5) + 1;
    NTCB_CUDA(cudaMemsetAsync(mask + w0, 0, sizeof(uint32_t) * (w1 - w0), ctx->side));
    prof_mark(ctx, 1, ctx->side);
    uint64_t cap = 0;
    ctx->prof.launches += launch_sample_set(ctx, ctx->side, mask, mode, r0, r1, cfg.c, root, 0, &cap);
    ctx->prof.launches += launch_sample_heavy(ctx, ctx->side, mask, mode, r0, r1, cfg.c, root, 0, cap);
    prof_end(ctx, ctx->side);
    NTCB_CUDA(cudaEventRecord(ctx->ev_sampled[mode][par], ctx->side));
  }
  return par;
}

// presampled >= 0: the parity enqueue_sample already filled for l = 0.
// Returns the entries this call will access (also added to the pending
// count that ntcb_collect hands back).
uint64_t enqueue_snmc(ntcb_context* ctx, int mode, uint64_t r0, uint64_t r1,
                      const ntcb_nmc_config& cfg, uint64_t rng_state, int presampled = -1,
                      bool y_set = false) {
  const uint64_t ld = ctx->ld;
  cudaStream_t st = ctx->stream;
  if (r1 <= r0) return 0;
  // A_0 = Y_0 = a_init (nmc.cpp:212-215); A already holds a_init (y_set: Y too).
  if (!y_set)
    NTCB_CUDA(cudaMemcpyAsync(ctx->Y[mode] + r0 * ld, ctx->A[mode] + r0 * ld,
                              sizeof(float) * (r1 - r0) * ld, cudaMemcpyDeviceToDevice, st));
  const DeviceView& v = ctx->views[mode];
  const uint64_t e0 = v.h_off[r0], e1 = v.h_off[r1];
  for (int l = 0; l < cfg.max_inner; ++l) {
    const int par = (l == 0 && presampled >= 0) ? presampled
                                                : enqueue_sample(ctx, mode, r0, r1, cfg, rng_state, l);
    uint32_t* mask = ctx->mask[mode][par];
    if (cfg.c < 1.0 && e1 > e0) NTCB_CUDA(cudaStreamWaitEvent(st, ctx->ev_sampled[mode][par], 0));
    prof_mark(ctx, 0, st);
    const int n = launch_update(ctx, mode, r0, r1, cfg, mask);
    ctx->prof.launches += n;
    ctx->prof.update_launches += n;
    prof_end(ctx, st);
    NTCB_CUDA(cudaEventRecord(ctx->ev_consumed[mode][par], st));
    ctx->consumed_valid[mode][par] = true;
  }
  host_of(ctx).queued = true;
  const uint64_t n = static_cast<uint64_t>(cfg.max_inner) * blocksize_sum(ctx, mode, r0, r1, cfg.c);
  host_of(ctx).pending_accessed += n;
  return n;
}

// Work whose count the caller consumes itself (s_nmc, ao_ntc): enqueued like
// any other, but its entries are taken out of the pending count again, so a
// later ntcb_collect still returns exactly the async work queued by the user.
uint64_t enqueue_snmc_owned(ntcb_context* ctx, int mode, uint64_t r0, uint64_t r1,
                            const ntcb_nmc_config& cfg, uint64_t rng_state, int presampled = -1,
                            bool y_set = false) {
  const uint64_t n = enqueue_snmc(ctx, mode, r0, r1, cfg, rng_state, presampled, y_set);
  host_of(ctx).pending_accessed -= n;
  return n;
}

// One AO iteration (every mode, Gauss-Seidel, ao.cpp:121-124) enqueued on the
// context's streams; returns its entries.  With ntcb_tuning.graph the sweep
// is captured into a CUDA graph (the side stream forked into the capture and
// joined back) and launched as one unit -- the graph exec is updated in place
// from sweep to sweep (same topology, new RNG roots and mask parities).  The
// first sweep of a context runs uncaptured: plans and buffers are allocated
// there, outside any capture.  Sweeps launched as graphs serialise on the
// stream, so their waits on the previous sweep's mask events are dropped.
uint64_t enqueue_sweep(ntcb_context* ctx, uint64_t k, const ntcb_nmc_config& cfg, uint64_t seed, bool owned) {
  HostState& hs = host_of(ctx);
  auto one = [&](int i) {
    const uint64_t st = fork64(fork64(fork64(seed, 2), k), static_cast<uint64_t>(i));  // ao.cpp:65-68
    return owned ? enqueue_snmc_owned(ctx, i, 0, ctx->dims[i], cfg, st) : enqueue_snmc(ctx, i, 0, ctx->dims[i], cfg, st);
  };
  uint64_t n = 0;
  if (!ctx->tune.graph || hs.sweep_warm != ctx->plan_epoch + 1 || ctx->prof.on) {
    for (int i = 0; i < ctx->order; ++i) n += one(i);
    hs.sweep_warm = ctx->plan_epoch + 1;  // plans of this epoch exist now
    return n;
  }
  if (!hs.ev_fork) NTCB_CUDA(cudaEventCreateWithFlags(&hs.ev_fork, cudaEventDisableTiming));
  if (!hs.ev_join) NTCB_CUDA(cudaEventCreateWithFlags(&hs.ev_join, cudaEventDisableTiming));
  for (auto& mm : ctx->consumed_valid) mm[0] = mm[1] = false;
  NTCB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  cudaGraph_t g = nullptr;
  try {
    NTCB_CUDA(cudaEventRecord(hs.ev_fork, ctx->stream));
    NTCB_CUDA(cudaStreamWaitEvent(ctx->side, hs.ev_fork, 0));
    for (int i = 0; i < ctx->order; ++i) n += one(i);
    NTCB_CUDA(cudaEventRecord(hs.ev_join, ctx->side));
    NTCB_CUDA(cudaStreamWaitEvent(ctx->stream, hs.ev_join, 0));
  } catch (...) {
    cudaStreamEndCapture(ctx->stream, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    throw;
  }
  NTCB_CUDA(cudaStreamEndCapture(ctx->stream, &g));
  if (hs.sweep_exec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(hs.sweep_exec, g, &info) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphExecDestroy(hs.sweep_exec);
      hs.sweep_exec = nullptr;
    }
  }
  if (!hs.sweep_exec) {
    const cudaError_t e = cudaGraphInstantiate(&hs.sweep_exec, g, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(g);
      NTCB_CUDA(e);
    }
  }
  cudaGraphDestroy(g);
  NTCB_CUDA(cudaGraphLaunch(hs.sweep_exec, ctx->stream));
  // later side-stream work (the next sweep's samples) starts after the graph;
  // the mask events recorded inside the capture are not waited on again
  NTCB_CUDA(cudaEventRecord(hs.ev_fork, ctx->stream));
  NTCB_CUDA(cudaStreamWaitEvent(ctx->side, hs.ev_fork, 0));
  for (auto& mm : ctx->consumed_valid) mm[0] = mm[1] = false;
  return n;
}

// Waits and converts a device-side row failure into the reference's exception.
// One host synchronisation: the main stream waits for the side stream, then
// the error key comes back by an async copy into pinned memory.  The pending
// entry count (async work queued through the C-ABI) is handed back and reset
// only when `accessed` is given: internal drains keep it for ntcb_collect.
void collect(ntcb_context* ctx, uint64_t* accessed) {
  NTCB_CUDA(cudaEventRecord(ctx->ev_side_done, ctx->side));
  NTCB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_side_done, 0));
  NTCB_CUDA(cudaMemcpyAsync(ctx->h_counters, ctx->counters, 2 * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, ctx->stream));
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
  auto& hs = host_of(ctx);
  hs.queued = false;
  const unsigned long long key = ctx->h_counters[1];
  const uint64_t pend = hs.pending_accessed;
  if (accessed) hs.pending_accessed = 0;
  if (key != ~0ull) {
    const unsigned long long reset = ~0ull;
    NTCB_CUDA(cudaMemcpyAsync(ctx->counters + 1, &reset, sizeof reset, cudaMemcpyHostToDevice, ctx->stream));
    NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
    const int mode = static_cast<int>(key >> 58);
    const uint64_t row = (key >> 2) & ((1ull << 56) - 1);
    const int kind = static_cast<int>(key & 3);
    hs.verified[mode] = false;
    if (kind == 0)
      fail(NTCB_ERUNTIME, "s_nmc: non-finite gradient at row " + std::to_string(row + 1) +
                              " (mode " + std::to_string(mode + 1) + ")");
    if (kind == 1) fail(NTCB_ERUNTIME, "power_method: non-finite entries in matrix");
    if (kind == 3) fail(NTCB_EINVAL, "s_nmc: a_init must be nonnegative");  // pinned-buffer path
    fail(NTCB_ERUNTIME, "row_step: step constant below lambda");
  }
  if (accessed) *accessed += pend;
}

float* host_stage(ntcb_context* ctx, uint64_t n) {
  auto& hs = host_of(ctx);
  if (hs.stage_n < n) {
    if (hs.stage) cudaFreeHost(hs.stage);
    hs.stage = nullptr;
    hs.stage_n = 0;
    NTCB_CUDA(cudaMallocHost(&hs.stage, sizeof(float) * n));
    hs.stage_n = n;
  }
  return hs.stage;
}

// A persistent host worker pool for the fp64 <-> fp32 factor conversions of
// the host-buffer entry points (spawning threads per call costs more than the
// conversion of a 10^4 x 20 factor).  Leaked on purpose: it must outlive any
// static destructor that could still run a conversion.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool();
    return *p;
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  // run f(t) for t in [0, n) (n <= size()); the caller runs t = 0
  void run(int n, const std::function<void(int)>& f) {
    if (n <= 1) {
      f(0);
      return;
    }
    {
      std::unique_lock<std::mutex> lk(m_);
      job_ = &f;
      jobs_ = n;
      next_ = 1;
      pending_ = n - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  HostPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned n = std::min(hw, 16u) - 1;
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    for (auto& w : workers_) w.detach();
  }
  void loop() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(m_);
    while (true) {
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      while (job_ && next_ < jobs_) {
        const int t = next_++;
        const std::function<void(int)>* f = job_;
        lk.unlock();
        (*f)(t);
        lk.lock();
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int jobs_ = 0, next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
};

// f(row_begin, row_end) over [0, rows), split over the pool for large
// factors (at most ntcb_tuning.host_threads threads when it is set)
template <class F>
bool parallel_rows(const ntcb_context* ctx, uint64_t rows, uint64_t per_row, F f) {
  HostPool& pool = HostPool::get();
  const uint64_t cap = ctx->tune.host_threads > 0 ? static_cast<uint64_t>(ctx->tune.host_threads) : pool.size();
  const uint64_t nt = std::min<uint64_t>(std::min<uint64_t>(pool.size(), cap),
                                         std::max<uint64_t>(1, rows * per_row / (1 << 15)));
  if (nt <= 1) return f(0, rows);
  std::vector<char> ok(nt, 1);
  const std::function<void(int)> job = [&](int t) {
    ok[t] = f(rows * t / nt, rows * (t + 1) / nt);
  };
  pool.run(static_cast<int>(nt), job);
  return std::all_of(ok.begin(), ok.end(), [](char c) { return c != 0; });
}

// host doubles -> pinned fp32 rows (ld stride, zero padding) -> async H2D on
// the main stream; false (nothing enqueued) when a value is negative or NaN
bool upload_factor_async(ntcb_context* ctx, float* dst, const double* src, uint64_t rows) {
  const uint64_t R = ctx->rank, ld = ctx->ld;
  float* tmp = host_stage(ctx, rows * ld);
  const bool ok = parallel_rows(ctx, rows, R, [&](uint64_t i0, uint64_t i1) {
    bool good = true;
    for (uint64_t i = i0; i < i1; ++i) {
      const double* s = src + i * R;
      float* d = tmp + i * ld;
      for (uint64_t r = 0; r < R; ++r) {
        good &= s[r] >= 0.0;
        d[r] = static_cast<float>(s[r]);
      }
      for (uint64_t r = R; r < ld; ++r) d[r] = 0.f;
    }
    return good;
  });
  if (!ok) return false;
  NTCB_CUDA(cudaMemcpyAsync(dst, tmp, sizeof(float) * rows * ld, cudaMemcpyHostToDevice, ctx->stream));
  return true;
}

// A and/or Y of `mode` -> pinned staging (async on the main stream)
void download_factors_enqueue(ntcb_context* ctx, int mode, bool a, bool y) {
  const uint64_t ld = ctx->ld, rows = ctx->dims[mode], n = rows * ld;
  float* tmp = host_stage(ctx, 2 * n);
  if (a) NTCB_CUDA(cudaMemcpyAsync(tmp, ctx->A[mode], sizeof(float) * n, cudaMemcpyDeviceToHost, ctx->stream));
  if (y) NTCB_CUDA(cudaMemcpyAsync(tmp + n, ctx->Y[mode], sizeof(float) * n, cudaMemcpyDeviceToHost, ctx->stream));
}

// staging -> host doubles (after the main stream has been synchronised)
void download_factors_finish(ntcb_context* ctx, int mode, double* a, double* y) {
  const uint64_t R = ctx->rank, ld = ctx->ld, rows = ctx->dims[mode], n = rows * ld;
  float* tmp = host_of(ctx).stage;
  parallel_rows(ctx, rows, 2 * R, [&](uint64_t i0, uint64_t i1) {
    for (int w = 0; w < 2; ++w) {
      double* dst = w ? y : a;
      if (!dst) continue;
      const float* src = tmp + w * n;
      for (uint64_t i = i0; i < i1; ++i)
        for (uint64_t r = 0; r < R; ++r) dst[i * R + r] = static_cast<double>(src[i * ld + r]);
    }
    return true;
  });
}

// A and/or Y of `mode` -> host doubles (one synchronisation)
void download_factors(ntcb_context* ctx, int mode, double* a, double* y) {
  download_factors_enqueue(ctx, mode, a != nullptr, y != nullptr);
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
  download_factors_finish(ctx, mode, a, y);
}

void upload_factor(ntcb_context* ctx, float* dst, const double* src, uint64_t rows) {
  const uint64_t R = ctx->rank, ld = ctx->ld;
  std::vector<float> tmp(rows * ld, 0.f);
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t r = 0; r < R; ++r) tmp[i * ld + r] = static_cast<float>(src[i * R + r]);
  NTCB_CUDA(cudaMemcpyAsync(dst, tmp.data(), sizeof(float) * rows * ld, cudaMemcpyHostToDevice,
                            ctx->stream));
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
}

void download_factor(ntcb_context* ctx, const float* src, double* dst, uint64_t rows) {
  const uint64_t R = ctx->rank, ld = ctx->ld;
  std::vector<float> tmp(rows * ld);
  NTCB_CUDA(cudaMemcpyAsync(tmp.data(), src, sizeof(float) * rows * ld, cudaMemcpyDeviceToHost,
                            ctx->stream));
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t r = 0; r < R; ++r) dst[i * R + r] = static_cast<double>(tmp[i * ld + r]);
}

bool all_nonneg(const double* p, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    if (!(p[i] >= 0.0)) return false;
  return true;
}

void free_factors(ntcb_context* ctx) {
  for (int m = 0; m < NTCB_MAX_ORDER; ++m) {
    if (ctx->A[m]) cudaFree(ctx->A[m]);
    if (ctx->Y[m]) cudaFree(ctx->Y[m]);
    ctx->A[m] = ctx->Y[m] = nullptr;
  }
  ctx->rank = ctx->ld = 0;
  ctx->nat_padded = false;
  drop_prefetch(ctx);
  for (int m = 0; m < NTCB_MAX_ORDER; ++m) ctx->n_peers[m] = 0;
}

void alloc_factors(ntcb_context* ctx, uint64_t rank) {
  if (rank == 0) fail(NTCB_EINVAL, "FactorSet: rank must be positive");
  if (rank > NTCB_MAX_RANK) fail(NTCB_EINVAL, "FactorSet: rank exceeds the supported maximum (64)");
  need_tensor(ctx);
  free_factors(ctx);
  ctx->rank = rank;
  // row stride: whole 32-byte sectors up to rank 31 (the tensor-core update
  // gathers feature blocks of 8), 16-byte multiples above
  ctx->ld = rank <= 31 ? (rank + 7) / 8 * 8 : (rank + 3) / 4 * 4;
  // nat_pad: 128-byte rows (one L1 line per gathered row) for the NAT update
  uint64_t fbytes = 0;
  for (int m = 0; m < ctx->order; ++m) fbytes += ctx->dims[m] * rank * 4;
  const bool pad = ctx->tune.nat_pad >= 1 || (ctx->tune.nat_pad == -1 && fbytes > (16ull << 20));
  ctx->nat_padded = pad && rank >= 9 && rank <= 24 && (ctx->order == 3 || ctx->order == 4);
  // ranks 9-16: 64-byte rows (four lanes per pick); 17-24: 128-byte rows
  if (ctx->nat_padded) ctx->ld = (rank <= 16 && ctx->tune.nat_pad != 2) ? 16 : 32;
  for (int m = 0; m < ctx->order; ++m) {
    // + 32 floats: the tensor-core gather of the last row may read past it
    const size_t bytes = sizeof(float) * (ctx->dims[m] * ctx->ld + 32);
    NTCB_CUDA(cudaMalloc(&ctx->A[m], bytes));
    NTCB_CUDA(cudaMalloc(&ctx->Y[m], bytes));
    NTCB_CUDA(cudaMemsetAsync(ctx->A[m], 0, bytes, ctx->stream));
    NTCB_CUDA(cudaMemsetAsync(ctx->Y[m], 0, bytes, ctx->stream));
  }
  for (auto& v : host_of(ctx).verified) v = false;
}

__global__ void k_uniform_factor(uint64_t root, uint64_t rows, int R, int ld, float* a, float* y) {
  const uint64_t n = rows * R;
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double v = static_cast<double>(mix64(root + (q + 1) * kGolden) >> 11) * 0x1.0p-53;
    const uint64_t i = q / R, r = q % R;
    a[i * ld + r] = static_cast<float>(v);
    y[i * ld + r] = static_cast<float>(v);
  }
}

// plateau (ao.cpp:21-26)
bool plateau(const std::vector<ntcb_metrics_record>& h, double tol) {
  if (h.size() < 4) return false;
  for (size_t t = h.size() - 3; t < h.size(); ++t)
    if (!(std::abs(h[t].rel_error - h[t - 1].rel_error) < tol)) return false;
  return true;
}

// ---- host-buffer S_NMC with page-locked caller buffers: the fp64 <-> fp32
// conversion runs on the device, the copies go straight between the caller's
// pinned arrays and the device (no host-side conversion or staging) ----------
__global__ void k_a_init_in(const double* src, uint64_t rows, int R, int ld, float* dst,
                            unsigned long long* counters, int mode) {
  const uint64_t n = rows * static_cast<uint64_t>(ld);
  bool bad = false;
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = q / ld;
    const int r = static_cast<int>(q - i * ld);
    float v = 0.f;
    if (r < R) {
      const double d = src[i * R + r];
      bad |= !(d >= 0.0);  // negative or NaN (nmc.cpp:202-210)
      v = static_cast<float>(d);
    }
    dst[q] = v;
  }
  // one key for the whole call: row 0, kind 3 ("a_init must be nonnegative")
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    atomicMin(&counters[1], (static_cast<unsigned long long>(mode) << 58) | 3ull);
}
// A = Y = a_init, only when every value passed (the update kernels see the
// error key and do nothing either: A and Y stay untouched, as in the reference)
__global__ void k_a_init_commit(const float* src, uint64_t n, float* A, float* Y, const unsigned long long* counters) {
  if (*reinterpret_cast<const volatile unsigned long long*>(&counters[1]) != ~0ull) return;
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float v = src[q];
    A[q] = v;
    Y[q] = v;
  }
}
__global__ void k_factors_out(const float* A, const float* Y, uint64_t rows, int R, int ld, double* a,
                              double* y) {
  const uint64_t n = rows * static_cast<uint64_t>(R);
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = q / R, r = q - i * R;
    if (a) a[q] = static_cast<double>(A[i * ld + r]);
    if (y) y[q] = static_cast<double>(Y[i * ld + r]);
  }
}

bool pinned(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

template <class T>
T* io_buffer(void*& buf, uint64_t& cap, uint64_t n) {
  if (cap < sizeof(T) * n) {
    if (buf) cudaFree(buf);
    buf = nullptr;
    cap = 0;
    NTCB_CUDA(cudaMalloc(&buf, sizeof(T) * n));
    cap = sizeof(T) * n;
  }
  return static_cast<T*>(buf);
}

}  // namespace

extern "C" {

const char* ntcb_last_error(void) { return g_err.c_str(); }
int ntcb_version(void) { return 1; }

int ntcb_create(int device, ntcb_context** out) {
  API_TRY
  if (!out) fail(NTCB_EINVAL, "ntcb_create: null out");
  int n = 0;
  NTCB_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) fail(NTCB_EINVAL, "ntcb_create: no such CUDA device");
  NTCB_CUDA(cudaSetDevice(device));
  auto* ctx = new ntcb_context();
  ctx->device = device;
  NTCB_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
  ctx->stream = ctx->own_stream;
  NTCB_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
  NTCB_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  for (auto& mm : ctx->ev_sampled)
    for (auto& e : mm) NTCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& mm : ctx->ev_consumed)
    for (auto& e : mm) NTCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  NTCB_CUDA(cudaEventCreateWithFlags(&ctx->ev_side_done, cudaEventDisableTiming));
  NTCB_CUDA(cudaMalloc(&ctx->counters, 8 * sizeof(unsigned long long)));
  NTCB_CUDA(cudaMallocHost(&ctx->h_counters, 8 * sizeof(unsigned long long)));
  const unsigned long long init[8] = {0, ~0ull, 0, 0, 0, 0, 0, 0};
  NTCB_CUDA(cudaMemcpy(ctx->counters, init, sizeof init, cudaMemcpyHostToDevice));
  for (auto& e : ctx->prof.ev) NTCB_CUDA(cudaEventCreate(&e));
  for (auto& e : ctx->prof.kev) NTCB_CUDA(cudaEventCreate(&e));
  ctx->host = new HostState();
  *out = ctx;
  API_CATCH
}

int ntcb_destroy(ntcb_context* ctx) {
  API_TRY
  if (!ctx) return NTCB_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  free_views(ctx);
  free_factors(ctx);
  if (ctx->red) cudaFree(ctx->red);
  cudaFree(ctx->counters);
  cudaFreeHost(ctx->h_counters);
  for (auto& e : ctx->prof.ev) cudaEventDestroy(e);
  for (auto& e : ctx->prof.kev) cudaEventDestroy(e);
  for (auto& mm : ctx->ev_sampled)
    for (auto& e : mm) cudaEventDestroy(e);
  for (auto& mm : ctx->ev_consumed)
    for (auto& e : mm) cudaEventDestroy(e);
  if (ctx->ev_side_done) cudaEventDestroy(ctx->ev_side_done);
  cudaStreamDestroy(ctx->side);
  cudaStreamDestroy(ctx->own_stream);
  if (host_of(ctx).stage) cudaFreeHost(host_of(ctx).stage);
  for (void* p : {host_of(ctx).io_in, host_of(ctx).io_f, host_of(ctx).io_out})
    if (p) cudaFree(p);
  if (host_of(ctx).sweep_exec) cudaGraphExecDestroy(host_of(ctx).sweep_exec);
  if (host_of(ctx).ev_fork) cudaEventDestroy(host_of(ctx).ev_fork);
  if (host_of(ctx).ev_join) cudaEventDestroy(host_of(ctx).ev_join);
  for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
  delete static_cast<HostState*>(ctx->host);
  delete ctx;
  API_CATCH
}

int ntcb_set_stream(ntcb_context* ctx, void* s) {
  API_TRY
  need_ctx(ctx);
  ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
  API_CATCH
}

int ntcb_synchronize(ntcb_context* ctx) {
  API_TRY
  need_ctx(ctx);
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_CATCH
}

void ntcb_tuning_defaults(ntcb_tuning* t) {
  if (t) *t = default_tuning();
}

int ntcb_set_tuning(ntcb_context* ctx, const ntcb_tuning* t) {
  API_TRY
  need_ctx(ctx);
  if (!t) fail(NTCB_EINVAL, "tuning: null");
  if (t->tc_p != 0 && t->tc_p != 4) fail(NTCB_EINVAL, "tuning: tc_p must be 0 or 4");
  if (t->update_wpc < 1 || t->update_wpc > 8) fail(NTCB_EINVAL, "tuning: update_wpc must be in [1, 8]");
  if (t->short_row < 0) fail(NTCB_EINVAL, "tuning: short_row must be >= 0");
  if (t->side_sampler_ctas < 0) fail(NTCB_EINVAL, "tuning: side_sampler_ctas must be >= 0");
  if (t->heavy_per < 1) fail(NTCB_EINVAL, "tuning: heavy_per must be >= 1");
  if (t->heavy_win_log2 < 16 || t->heavy_win_log2 > 30 || t->heavy_big_log2 < 16 || t->heavy_big_log2 > 30)
    fail(NTCB_EINVAL, "tuning: heavy_win_log2 / heavy_big_log2 must be in [16, 30]");
  if (t->host_threads < 0) fail(NTCB_EINVAL, "tuning: host_threads must be >= 0");
  if (t->nat_pad < -1 || t->nat_pad > 2) fail(NTCB_EINVAL, "tuning: nat_pad must be -1, 0, 1 or 2");
  if (t->peer_fence < 0 || t->peer_fence > 2) fail(NTCB_EINVAL, "tuning: peer_fence must be 0, 1 or 2");
  if (t->graph != 0 && t->graph != 1) fail(NTCB_EINVAL, "tuning: graph must be 0 or 1");
  if (t->tiny_sampler != 0 && t->tiny_sampler != 1) fail(NTCB_EINVAL, "tuning: tiny_sampler must be 0 or 1");
  if (t->item_order != 0 && t->item_order != 1) fail(NTCB_EINVAL, "tuning: item_order must be 0 or 1");
  if (t->update_ctas_per_sm < 0) fail(NTCB_EINVAL, "tuning: update_ctas_per_sm must be >= 0");
  if (t->update_carveout < -1 || t->update_carveout > 100)
    fail(NTCB_EINVAL, "tuning: update_carveout must be -1 or a percentage");
  collect(ctx, nullptr);  // queued work keeps the plans it was launched with
  drop_prefetch(ctx);
  ctx->tune = *t;
  drop_plans(ctx);  // plans bake in the heavy-window sizes and the short-row decision
  drop_heavy(ctx);
  drop_sample_plans(ctx);
  API_CATCH
}

int ntcb_get_tuning(ntcb_context* ctx, ntcb_tuning* t) {
  API_TRY
  need_ctx(ctx);
  if (!t) fail(NTCB_EINVAL, "tuning: null");
  *t = ctx->tune;
  API_CATCH
}

int ntcb_host_alloc(uint64_t bytes, void** out) {
  API_TRY
  if (!out) fail(NTCB_EINVAL, "host_alloc: null out");
  *out = nullptr;
  NTCB_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
  API_CATCH
}

int ntcb_host_free(void* p) {
  API_TRY
  if (p) NTCB_CUDA(cudaFreeHost(p));
  API_CATCH
}

uint64_t ntcb_rng_fork(uint64_t state, uint64_t tag) { return fork64(state, tag); }
uint64_t ntcb_sweep_stream_state(uint64_t seed, uint64_t sweep, int mode) {
  return fork64(fork64(fork64(seed, 2), sweep), static_cast<uint64_t>(mode));  // ao.cpp:65-68
}

int ntcb_tensor_load(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                     const uint32_t* indices, const double* values) {
  API_TRY
  need_ctx(ctx);
  free_factors(ctx);
  load_tensor_f64(ctx, order, dims, nnz, indices, values);
  host_of(ctx).bs_cache.clear();
  API_CATCH
}

int ntcb_tensor_load_f32(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                         const uint32_t* indices, const float* values) {
  API_TRY
  need_ctx(ctx);
  free_factors(ctx);
  load_tensor_f32(ctx, order, dims, nnz, indices, values, false);
  host_of(ctx).bs_cache.clear();
  API_CATCH
}

int ntcb_tensor_load_device(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                            const uint32_t* d_indices, const float* d_values) {
  API_TRY
  need_ctx(ctx);
  free_factors(ctx);
  load_tensor_f32(ctx, order, dims, nnz, d_indices, d_values, true);
  host_of(ctx).bs_cache.clear();
  API_CATCH
}

int ntcb_synth_uniform(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                       uint64_t true_rank, double sigma, uint64_t seed) {
  API_TRY
  need_ctx(ctx);
  free_factors(ctx);
  synth_uniform(ctx, order, dims, nnz, true_rank, sigma, seed);
  host_of(ctx).bs_cache.clear();
  API_CATCH
}

int ntcb_synth(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
               uint64_t true_rank, double sigma, uint64_t seed, const double* zipf_alpha,
               int value_kind) {
  API_TRY
  need_ctx(ctx);
  free_factors(ctx);
  synth_general(ctx, order, dims, nnz, true_rank, sigma, seed, zipf_alpha, value_kind);
  host_of(ctx).bs_cache.clear();
  API_CATCH
}

int ntcb_tensor_read_tns(ntcb_context* ctx, const char* path) {
  API_TRY
  need_ctx(ctx);
  int order = 0;
  uint64_t dims[NTCB_MAX_ORDER] = {};
  uint64_t nnz = 0;
  uint32_t* idx = nullptr;
  double* val = nullptr;
  const int rc = ntcb_tns_parse(path, &order, dims, &nnz, &idx, &val);
  if (rc) fail(rc, ntcb_tns_last_error());
  struct Free {
    void* a;
    void* b;
    ~Free() {
      ntcb_free(a);
      ntcb_free(b);
    }
  } fr{idx, val};
  free_factors(ctx);
  load_tensor_f64(ctx, order, dims, nnz, idx, val);
  host_of(ctx).bs_cache.clear();
  API_CATCH
}

int ntcb_tensor_info(ntcb_context* ctx, int* order, uint64_t* dims, uint64_t* nnz) {
  API_TRY
  need_ctx(ctx);
  if (order) *order = ctx->order;
  if (dims)
    for (int m = 0; m < ctx->order; ++m) dims[m] = ctx->dims[m];
  if (nnz) *nnz = ctx->nnz;
  API_CATCH
}

int ntcb_view_export(ntcb_context* ctx, int mode, uint64_t* offsets, uint32_t* others,
                     float* values) {
  API_TRY
  need_ctx(ctx);
  need_tensor(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "view_export: mode out of range");
  if (others || values) need_rows(ctx, mode, 0, ctx->dims[mode]);
  const DeviceView& v = ctx->views[mode];
  const uint64_t nnz = ctx->nnz;
  const int no = ctx->order - 1;
  if (offsets) std::memcpy(offsets, v.h_off, sizeof(uint64_t) * (v.rows + 1));
  if (others && nnz) {
    std::vector<uint32_t> col(nnz);
    for (int k = 0; k < no; ++k) {
      NTCB_CUDA(cudaMemcpy(col.data(), v.oth[k], sizeof(uint32_t) * nnz, cudaMemcpyDeviceToHost));
      for (uint64_t t = 0; t < nnz; ++t) others[t * no + k] = col[t];
    }
  }
  if (values && nnz)
    NTCB_CUDA(cudaMemcpy(values, v.val, sizeof(float) * nnz, cudaMemcpyDeviceToHost));
  API_CATCH
}

int ntcb_view_export_rows(ntcb_context* ctx, int mode, uint64_t row_begin, uint64_t row_end,
                          uint64_t* offsets, uint32_t* others, float* values) {
  API_TRY
  need_ctx(ctx);
  need_tensor(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "view_export: mode out of range");
  const DeviceView& v = ctx->views[mode];
  if (row_begin > row_end || row_end > v.rows) fail(NTCB_ERANGE, "view_export: rows out of range");
  if (others || values) need_rows(ctx, mode, row_begin, row_end);
  const uint64_t e0 = v.h_off[row_begin], e1 = v.h_off[row_end], n = e1 - e0;
  const int no = ctx->order - 1;
  if (offsets) std::memcpy(offsets, v.h_off + row_begin, sizeof(uint64_t) * (row_end - row_begin + 1));
  if (others && n) {
    std::vector<uint32_t> col(n);
    for (int k = 0; k < no; ++k) {
      NTCB_CUDA(cudaMemcpy(col.data(), v.oth[k] + e0, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
      for (uint64_t t = 0; t < n; ++t) others[t * no + k] = col[t];
    }
  }
  if (values && n) NTCB_CUDA(cudaMemcpy(values, v.val + e0, sizeof(float) * n, cudaMemcpyDeviceToHost));
  API_CATCH
}

int ntcb_tensor_export(ntcb_context* ctx, uint32_t* indices, float* values) {
  API_TRY
  need_ctx(ctx);
  need_tensor(ctx);
  need_rows(ctx, 0, 0, ctx->dims[0]);
  // the mode-0 view IS the canonical lexicographic order (mode_view.cpp:5-7)
  const DeviceView& v = ctx->views[0];
  const uint64_t nnz = ctx->nnz;
  const int N = ctx->order;
  if (indices && nnz) {
    std::vector<uint32_t> col(nnz);
    for (int k = 0; k < N - 1; ++k) {
      NTCB_CUDA(cudaMemcpy(col.data(), v.oth[k], sizeof(uint32_t) * nnz, cudaMemcpyDeviceToHost));
      for (uint64_t t = 0; t < nnz; ++t) indices[t * N + k + 1] = col[t];
    }
    for (uint64_t p = 0; p < v.rows; ++p)
      for (uint64_t t = v.h_off[p]; t < v.h_off[p + 1]; ++t) indices[t * N] = static_cast<uint32_t>(p);
  }
  if (values && nnz)
    NTCB_CUDA(cudaMemcpy(values, v.val, sizeof(float) * nnz, cudaMemcpyDeviceToHost));
  API_CATCH
}

int ntcb_view_keep_rows(ntcb_context* ctx, int mode, uint64_t row_begin, uint64_t row_end) {
  API_TRY
  need_ctx(ctx);
  need_tensor(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "view_keep_rows: mode out of range");
  if (row_begin > row_end || row_end > ctx->dims[mode]) fail(NTCB_ERANGE, "view_keep_rows: rows out of range");
  need_rows(ctx, mode, row_begin, row_end);
  collect(ctx, nullptr);
  NTCB_CUDA(cudaStreamSynchronize(ctx->side));
  drop_prefetch(ctx);
  DeviceView& v = ctx->views[mode];
  const int no = ctx->order - 1;
  const uint64_t e0 = v.h_off[row_begin], e1 = v.h_off[row_end];
  const uint64_t a_lo = e0 & ~uint64_t(31);  // whole 128-byte batches stay in bounds
  const uint64_t n = e1 - a_lo + kViewPad;
  for (int k = 0; k < no; ++k) {
    uint32_t* nb = nullptr;
    NTCB_CUDA(cudaMalloc(&nb, sizeof(uint32_t) * n));
    NTCB_CUDA(cudaMemcpy(nb, v.oth[k] + a_lo, sizeof(uint32_t) * (e1 - a_lo), cudaMemcpyDeviceToDevice));
    NTCB_CUDA(cudaMemset(nb + (e1 - a_lo), 0, sizeof(uint32_t) * kViewPad));
    NTCB_CUDA(cudaFree(v.oth[k] + v.a_lo));
    v.oth[k] = nb - a_lo;
  }
  {
    float* nb = nullptr;
    NTCB_CUDA(cudaMalloc(&nb, sizeof(float) * n));
    NTCB_CUDA(cudaMemcpy(nb, v.val + a_lo, sizeof(float) * (e1 - a_lo), cudaMemcpyDeviceToDevice));
    NTCB_CUDA(cudaMemset(nb + (e1 - a_lo), 0, sizeof(float) * kViewPad));
    NTCB_CUDA(cudaFree(v.val + v.a_lo));
    v.val = nb - a_lo;
  }
  const uint64_t words = (e1 - a_lo) / 32 + 2 + kViewPad / 32;
  for (int q = 0; q < 2; ++q) {
    uint32_t* nb = nullptr;
    NTCB_CUDA(cudaMalloc(&nb, sizeof(uint32_t) * words));
    NTCB_CUDA(cudaMemset(nb, 0, sizeof(uint32_t) * words));
    NTCB_CUDA(cudaFree(ctx->mask[mode][q] + (v.a_lo >> 5)));
    ctx->mask[mode][q] = nb - (a_lo >> 5);
    ctx->consumed_valid[mode][q] = false;
  }
  v.a_lo = a_lo;
  v.row_lo = row_begin;
  v.row_hi = row_end;
  uint64_t mx = 0;
  for (uint64_t p = row_begin; p < row_end; ++p) mx = std::max(mx, v.h_off[p + 1] - v.h_off[p]);
  v.max_slice = mx;
  // the per-entry sampler scratch covers the largest resident slab
  if (ctx->perm_scratch) {
    uint64_t need = 0;
    for (int m = 0; m < ctx->order; ++m) {
      const DeviceView& w = ctx->views[m];
      need = std::max(need, w.h_off[w.row_hi] - w.a_lo + kViewPad);
    }
    if (need < ctx->perm_scratch_n) {
      uint32_t* ns = nullptr;
      NTCB_CUDA(cudaMalloc(&ns, sizeof(uint32_t) * need));
      NTCB_CUDA(cudaFree(ctx->perm_scratch));
      ctx->perm_scratch = ns;
      ctx->perm_scratch_n = need;
    }
  }
  drop_plans(ctx);
  drop_heavy(ctx);
  drop_sample_plans(ctx);
  drop_metric_plans(ctx);
  host_of(ctx).bs_cache.clear();
  API_CATCH
}

int ntcb_view_resident(ntcb_context* ctx, int mode, uint64_t* row_begin, uint64_t* row_end,
                       uint64_t* device_bytes) {
  API_TRY
  need_ctx(ctx);
  need_tensor(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "view_resident: mode out of range");
  const DeviceView& v = ctx->views[mode];
  if (row_begin) *row_begin = v.row_lo;
  if (row_end) *row_end = v.row_hi;
  if (device_bytes) {
    const uint64_t n = v.h_off[v.row_hi] - v.a_lo + kViewPad;
    *device_bytes = n * 4 * static_cast<uint64_t>(ctx->order) + sizeof(uint64_t) * (v.rows + 1) +
                    2 * sizeof(uint32_t) * (n / 32 + 2);
  }
  API_CATCH
}

int ntcb_factors_init(ntcb_context* ctx, uint64_t rank, const double* const* factors,
                      const double* const* momentum) {
  API_TRY
  need_ctx(ctx);
  alloc_factors(ctx, rank);
  auto& hs = host_of(ctx);
  for (int m = 0; m < ctx->order; ++m) {
    upload_factor(ctx, ctx->A[m], factors[m], ctx->dims[m]);
    upload_factor(ctx, ctx->Y[m], momentum ? momentum[m] : factors[m], ctx->dims[m]);
    hs.verified[m] = all_nonneg(factors[m], ctx->dims[m] * rank);
  }
  API_CATCH
}

int ntcb_factors_random(ntcb_context* ctx, uint64_t rank, uint64_t seed) {
  API_TRY
  need_ctx(ctx);
  alloc_factors(ctx, rank);
  const uint64_t base = fork64(seed, 1);  // initial_factors, ao.cpp:70-73
  for (int m = 0; m < ctx->order; ++m) {
    const uint64_t n = ctx->dims[m] * rank;
    const unsigned g = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 4096));
    k_uniform_factor<<<g, 256, 0, ctx->stream>>>(fork64(base, m), ctx->dims[m],
                                                 static_cast<int>(rank), static_cast<int>(ctx->ld),
                                                 ctx->A[m], ctx->Y[m]);
    NTCB_CUDA(cudaGetLastError());
    host_of(ctx).verified[m] = true;
  }
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_CATCH
}

int ntcb_factor_set(ntcb_context* ctx, int mode, const double* a, const double* y) {
  API_TRY
  need_ctx(ctx);
  need_factors(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "factor_set: mode out of range");
  if (a) {
    upload_factor(ctx, ctx->A[mode], a, ctx->dims[mode]);
    host_of(ctx).verified[mode] = all_nonneg(a, ctx->dims[mode] * ctx->rank);
  }
  if (y) upload_factor(ctx, ctx->Y[mode], y, ctx->dims[mode]);
  API_CATCH
}

int ntcb_factor_get(ntcb_context* ctx, int mode, double* a, double* y) {
  API_TRY
  need_ctx(ctx);
  need_factors(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "factor_get: mode out of range");
  download_factors(ctx, mode, a, y);
  API_CATCH
}

int ntcb_factor_ipc_handle(ntcb_context* ctx, int mode, void* handle64) {
  API_TRY
  need_ctx(ctx);
  need_factors(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "factor_ipc_handle: mode out of range");
  if (!handle64) fail(NTCB_EINVAL, "factor_ipc_handle: null output");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "64-byte IPC handle");
  cudaIpcMemHandle_t h;
  NTCB_CUDA(cudaIpcGetMemHandle(&h, ctx->A[mode]));
  std::memcpy(handle64, &h, sizeof h);
  API_CATCH
}

int ntcb_ipc_open(ntcb_context* ctx, const void* handle64, void** ptr) {
  API_TRY
  need_ctx(ctx);
  if (!handle64 || !ptr) fail(NTCB_EINVAL, "ipc_open: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof h);
  void* p = nullptr;
  NTCB_CUDA(cudaSetDevice(ctx->device));
  NTCB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  ctx->ipc_opened.push_back(p);
  *ptr = p;
  API_CATCH
}

int ntcb_factor_set_peers(ntcb_context* ctx, int mode, int n, void* const* peer_ptrs) {
  API_TRY
  need_ctx(ctx);
  need_factors(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "factor_set_peers: mode out of range");
  if (n < 0 || n > 7) fail(NTCB_EINVAL, "factor_set_peers: at most 7 peers");
  if (n > 0 && !peer_ptrs) fail(NTCB_EINVAL, "factor_set_peers: null pointer array");
  collect(ctx, nullptr);  // no queued update may still use the old peer set
  for (int q = 0; q < 7; ++q) ctx->peerA[mode][q] = q < n ? static_cast<float*>(peer_ptrs[q]) : nullptr;
  ctx->n_peers[mode] = n;
  API_CATCH
}

int ntcb_factor_device_ptr(ntcb_context* ctx, int mode, int which, void** ptr, uint64_t* ld) {
  API_TRY
  need_ctx(ctx);
  need_factors(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "factor_device_ptr: mode out of range");
  if (ptr) *ptr = which ? ctx->Y[mode] : ctx->A[mode];
  if (ld) *ld = ctx->ld;
  API_CATCH
}

// ntcb_s_nmc / ntcb_s_nmc_host: the host-buffer form enqueues the copies of
// the updated factor and momentum before the call's single synchronisation
// The prefetched sampled set of (mode, c, rng_state), if there is one: its
// mask parity (the buffer stays reserved until the update has consumed it).
static int take_prefetch(ntcb_context* ctx, int mode, const ntcb_nmc_config& cfg, uint64_t rng_state) {
  auto& p = host_of(ctx).prefetch[mode];
  if (!p.valid || p.rng_state != rng_state || p.c != cfg.c) return -1;
  p.valid = false;
  return p.parity;
}
static int sample_first(ntcb_context* ctx, int mode, const ntcb_nmc_config& cfg, uint64_t rng_state) {
  const int pre = take_prefetch(ctx, mode, cfg, rng_state);
  return pre >= 0 ? pre : enqueue_sample(ctx, mode, 0, ctx->dims[mode], cfg, rng_state, 0);
}

static int s_nmc_impl(ntcb_context* ctx, int mode, const double* a_init, double* a_out, double* y_out,
                      bool outs, const ntcb_nmc_config* cfg, uint64_t rng_state, uint64_t* entries_accessed) {
  API_TRY
  need_ctx(ctx);
  validate_nmc(cfg);
  need_factors(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_EINVAL, "s_nmc: mode out of range");
  need_rows(ctx, mode, 0, ctx->dims[mode]);
  auto& hs = host_of(ctx);
  if (!a_init && !hs.verified[mode]) fail(NTCB_EINVAL, "s_nmc: a_init must be nonnegative");
  if (hs.queued) collect(ctx, nullptr);  // drain (and report) anything queued before
  int pre = -1;
  const uint64_t rows = ctx->dims[mode], R = ctx->rank, ld = ctx->ld;
  const bool dev_io = a_init && pinned(a_init) && (!outs || ((!a_out || pinned(a_out)) && (!y_out || pinned(y_out))));
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>((rows * ld + 255) / 256, 8ull * ctx->sm_count));
  if (dev_io) {
    // page-locked caller buffers: a_init goes to the device as fp64 and is
    // checked and converted there; no host work on the critical path
    if (cfg->max_inner > 0) pre = sample_first(ctx, mode, *cfg, rng_state);
    HostState& h = hs;
    double* din = io_buffer<double>(h.io_in, h.io_in_cap, rows * R);
    float* dsc = io_buffer<float>(h.io_f, h.io_f_cap, rows * ld);
    NTCB_CUDA(cudaMemcpyAsync(din, a_init, sizeof(double) * rows * R, cudaMemcpyHostToDevice, ctx->stream));
    k_a_init_in<<<g, 256, 0, ctx->stream>>>(din, rows, static_cast<int>(R), static_cast<int>(ld), dsc, ctx->counters,
                                           mode);
    k_a_init_commit<<<g, 256, 0, ctx->stream>>>(dsc, rows * ld, ctx->A[mode], ctx->Y[mode], ctx->counters);
    NTCB_CUDA(cudaGetLastError());
    const uint64_t own = enqueue_snmc_owned(ctx, mode, 0, rows, *cfg, rng_state, pre, true);
    if (outs && (a_out || y_out)) {
      double* dout = io_buffer<double>(h.io_out, h.io_out_cap, 2 * rows * R);
      k_factors_out<<<g, 256, 0, ctx->stream>>>(ctx->A[mode], ctx->Y[mode], rows, static_cast<int>(R),
                                               static_cast<int>(ld), a_out ? dout : nullptr,
                                               y_out ? dout + rows * R : nullptr);
      NTCB_CUDA(cudaGetLastError());
      if (a_out)
        NTCB_CUDA(cudaMemcpyAsync(a_out, dout, sizeof(double) * rows * R, cudaMemcpyDeviceToHost, ctx->stream));
      if (y_out)
        NTCB_CUDA(cudaMemcpyAsync(y_out, dout + rows * R, sizeof(double) * rows * R, cudaMemcpyDeviceToHost,
                                  ctx->stream));
    }
    collect(ctx, nullptr);  // the one synchronisation; a_init errors surface here
    hs.verified[mode] = true;
    if (entries_accessed) *entries_accessed += own;
    return NTCB_OK;
  }
  if (a_init) {
    // the first sample does not read factors: it runs on the side stream
    // while a_init is converted and copied in
    if (cfg->max_inner > 0) pre = sample_first(ctx, mode, *cfg, rng_state);
    if (!upload_factor_async(ctx, ctx->A[mode], a_init, ctx->dims[mode])) {
      hs.verified[mode] = false;
      collect(ctx, nullptr);
      fail(NTCB_EINVAL, "s_nmc: a_init must be nonnegative");
    }
    hs.verified[mode] = true;
  }
  if (!a_init && cfg->max_inner > 0) pre = take_prefetch(ctx, mode, *cfg, rng_state);
  const uint64_t own = enqueue_snmc_owned(ctx, mode, 0, ctx->dims[mode], *cfg, rng_state, pre);
  if (outs) download_factors_enqueue(ctx, mode, a_out != nullptr, y_out != nullptr);
  collect(ctx, nullptr);  // the one synchronisation of the call
  if (entries_accessed) *entries_accessed += own;  // nmc.cpp:270 (+=)
  if (outs) download_factors_finish(ctx, mode, a_out, y_out);
  API_CATCH
}

int ntcb_s_nmc(ntcb_context* ctx, int mode, const double* a_init, const ntcb_nmc_config* cfg,
               uint64_t rng_state, uint64_t* entries_accessed) {
  return s_nmc_impl(ctx, mode, a_init, nullptr, nullptr, false, cfg, rng_state, entries_accessed);
}

int ntcb_s_nmc_host(ntcb_context* ctx, int mode, const double* a_init, double* a_out,
                    double* y_out, const ntcb_nmc_config* cfg, uint64_t rng_state,
                    uint64_t* entries_accessed) {
  return s_nmc_impl(ctx, mode, a_init, a_out, y_out, true, cfg, rng_state, entries_accessed);
}

int ntcb_sample_prefetch(ntcb_context* ctx, int mode, const ntcb_nmc_config* cfg, uint64_t rng_state) {
  API_TRY
  need_ctx(ctx);
  validate_nmc(cfg);
  need_tensor(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_EINVAL, "s_nmc: mode out of range");
  need_rows(ctx, mode, 0, ctx->dims[mode]);
  if (cfg->max_inner < 1 || cfg->c >= 1.0) return NTCB_OK;  // nothing is drawn (c = 1 consumes no randomness)
  auto& p = host_of(ctx).prefetch[mode];
  const int par = enqueue_sample(ctx, mode, 0, ctx->dims[mode], *cfg, rng_state, 0);  // clears p.valid
  p.valid = true;
  p.rng_state = rng_state;
  p.c = cfg->c;
  p.parity = par;
  // `queued` stays as it is: the matching s_nmc call must not drain the sampler first
  // (every entry point that frees or replaces device state collects unconditionally)
  API_CATCH
}

int ntcb_s_nmc_rows_async(ntcb_context* ctx, int mode, uint64_t row_begin, uint64_t row_end,
                          const ntcb_nmc_config* cfg, uint64_t rng_state) {
  API_TRY
  need_ctx(ctx);
  validate_nmc(cfg);
  need_factors(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_EINVAL, "s_nmc: mode out of range");
  if (row_begin > row_end || row_end > ctx->dims[mode])
    fail(NTCB_ERANGE, "s_nmc: row range out of bounds");
  need_rows(ctx, mode, row_begin, row_end);
  if (!host_of(ctx).verified[mode]) fail(NTCB_EINVAL, "s_nmc: a_init must be nonnegative");
  enqueue_snmc(ctx, mode, row_begin, row_end, *cfg, rng_state);
  API_CATCH
}

int ntcb_segment_length(ntcb_context* ctx, int mode, uint64_t* seg) {
  API_TRY
  need_ctx(ctx);
  need_tensor(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "segment_length: mode out of range");
  if (seg) *seg = segment_length(ctx, mode);
  API_CATCH
}

int ntcb_s_nmc_chunks_async(ntcb_context* ctx, int mode, uint64_t row, uint32_t chunk_begin,
                            uint32_t chunk_end, const ntcb_nmc_config* cfg, uint64_t rng_state, void* d_slots) {
  API_TRY
  need_ctx(ctx);
  validate_nmc(cfg);
  need_factors(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_EINVAL, "s_nmc: mode out of range");
  if (row >= ctx->dims[mode]) fail(NTCB_ERANGE, "s_nmc_chunks: row out of range");
  need_rows(ctx, mode, row, row + 1);
  if (cfg->max_inner != 1) fail(NTCB_EINVAL, "s_nmc_chunks: a shared row needs max_inner = 1");
  if (!d_slots) fail(NTCB_EINVAL, "s_nmc_chunks: null slot buffer");
  if (!host_of(ctx).verified[mode]) fail(NTCB_EINVAL, "s_nmc: a_init must be nonnegative");
  const int par = enqueue_sample(ctx, mode, row, row + 1, *cfg, rng_state, 0);
  const DeviceView& v = ctx->views[mode];
  if (cfg->c < 1.0 && v.h_off[row + 1] > v.h_off[row])
    NTCB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_sampled[mode][par], 0));
  ctx->prof.launches += launch_update_chunks(ctx, mode, row, chunk_begin, chunk_end, *cfg, ctx->mask[mode][par],
                                             static_cast<float*>(d_slots));
  NTCB_CUDA(cudaEventRecord(ctx->ev_consumed[mode][par], ctx->stream));
  ctx->consumed_valid[mode][par] = true;
  host_of(ctx).queued = true;
  API_CATCH
}

int ntcb_finalize_row_async(ntcb_context* ctx, int mode, uint64_t row, const void* d_slots, uint32_t nslots,
                            const ntcb_nmc_config* cfg) {
  API_TRY
  need_ctx(ctx);
  validate_nmc(cfg);
  need_factors(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_EINVAL, "s_nmc: mode out of range");
  if (row >= ctx->dims[mode]) fail(NTCB_ERANGE, "finalize_row: row out of range");
  if (cfg->max_inner != 1) fail(NTCB_EINVAL, "s_nmc_chunks: a shared row needs max_inner = 1");
  if (!d_slots) fail(NTCB_EINVAL, "finalize_row: null slot buffer");
  const uint64_t n = ctx->views[mode].h_off[row + 1] - ctx->views[mode].h_off[row];
  const uint64_t seg = segment_length(ctx, mode);
  if (nslots != (n + seg - 1) / seg) fail(NTCB_EINVAL, "finalize_row: slot count differs from the row's chunks");
  const uint64_t b = blocksize_for(cfg->c, n);
  if (b > 0) ctx->prof.launches += launch_finalize_row(ctx, mode, row, static_cast<const float*>(d_slots), nslots, *cfg);
  host_of(ctx).pending_accessed += b;  // nmc.cpp:238, counted once (by the row's owner)
  host_of(ctx).queued = true;
  API_CATCH
}

int ntcb_collect(ntcb_context* ctx, uint64_t* entries_accessed) {
  API_TRY
  need_ctx(ctx);
  collect(ctx, entries_accessed);
  API_CATCH
}

int ntcb_sample_rows(ntcb_context* ctx, int mode, double c, uint64_t rng_state, uint64_t l,
                     uint64_t row_begin, uint64_t row_end, uint64_t* pick_offsets,
                     uint32_t* picks) {
  API_TRY
  need_ctx(ctx);
  need_tensor(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "sample_rows: mode out of range");
  if (row_begin > row_end || row_end > ctx->dims[mode])
    fail(NTCB_ERANGE, "sample_row: row out of range");
  if (!(c > 0.0 && c <= 1.0)) fail(NTCB_EINVAL, "sample_row: c must be in (0, 1]");
  need_rows(ctx, mode, row_begin, row_end);
  const uint64_t* off = ctx->views[mode].h_off;
  const uint64_t rows = row_end - row_begin;
  std::vector<uint64_t> po(rows + 1, 0);
  for (uint64_t i = 0; i < rows; ++i)
    po[i + 1] = po[i] + blocksize_for(c, off[row_begin + i + 1] - off[row_begin + i]);
  if (pick_offsets) std::memcpy(pick_offsets, po.data(), sizeof(uint64_t) * (rows + 1));
  if (!picks || po[rows] == 0) return NTCB_OK;
  uint64_t* d_po = nullptr;
  uint32_t* d_pk = nullptr;
  NTCB_CUDA(cudaMalloc(&d_po, sizeof(uint64_t) * (rows + 1)));
  NTCB_CUDA(cudaMalloc(&d_pk, sizeof(uint32_t) * po[rows]));
  NTCB_CUDA(cudaMemcpy(d_po, po.data(), sizeof(uint64_t) * (rows + 1), cudaMemcpyHostToDevice));
  collect(ctx, nullptr);
  host_of(ctx).prefetch[mode].valid = false;  // mask buffer 0 is overwritten below
  uint32_t* mask = ctx->mask[mode][0];
  const uint64_t e0 = off[row_begin], e1 = off[row_end];
  if (e1 > e0) {
    const uint64_t w0 = e0 >> 5, w1 = ((e1 - 1) >> 5) + 1;
    NTCB_CUDA(cudaMemsetAsync(mask + w0, 0, sizeof(uint32_t) * (w1 - w0), ctx->stream));
  }
  launch_sample(ctx, ctx->stream, mask, mode, row_begin, row_end, c, fork64(rng_state, l), d_pk, d_po);
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
  NTCB_CUDA(cudaMemcpy(picks, d_pk, sizeof(uint32_t) * po[rows], cudaMemcpyDeviceToHost));
  cudaFree(d_po);
  cudaFree(d_pk);
  API_CATCH
}

int ntcb_sample_row(ntcb_context* ctx, int mode, uint64_t row, double c, uint64_t row_state,
                    uint32_t* picks, uint64_t* count) {
  API_TRY
  need_ctx(ctx);
  need_tensor(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "sample_row: mode out of range");
  if (row >= ctx->dims[mode]) fail(NTCB_ERANGE, "sample_row: row out of range");
  if (!(c > 0.0 && c <= 1.0)) fail(NTCB_EINVAL, "sample_row: c must be in (0, 1]");
  need_rows(ctx, mode, row, row + 1);
  const uint64_t* off = ctx->views[mode].h_off;
  const uint64_t b = blocksize_for(c, off[row + 1] - off[row]);
  if (count) *count = b;
  if (!picks || b == 0) return NTCB_OK;
  uint64_t* d_po = nullptr;
  uint32_t* d_pk = nullptr;
  const uint64_t po[2] = {0, b};
  NTCB_CUDA(cudaMalloc(&d_po, sizeof po));
  NTCB_CUDA(cudaMalloc(&d_pk, sizeof(uint32_t) * b));
  NTCB_CUDA(cudaMemcpy(d_po, po, sizeof po, cudaMemcpyHostToDevice));
  collect(ctx, nullptr);
  host_of(ctx).prefetch[mode].valid = false;  // mask buffer 0 is overwritten below
  uint32_t* mask = ctx->mask[mode][0];
  const uint64_t e0 = off[row], e1 = off[row + 1];
  const uint64_t w0 = e0 >> 5, w1 = ((e1 - 1) >> 5) + 1;
  NTCB_CUDA(cudaMemsetAsync(mask + w0, 0, sizeof(uint32_t) * (w1 - w0), ctx->stream));
  launch_sample(ctx, ctx->stream, mask, mode, row, row + 1, c, row_state, d_pk, d_po, 1);
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
  NTCB_CUDA(cudaMemcpy(picks, d_pk, sizeof(uint32_t) * b, cudaMemcpyDeviceToHost));
  cudaFree(d_po);
  cudaFree(d_pk);
  API_CATCH
}

int ntcb_sample_mask(ntcb_context* ctx, int mode, double c, uint64_t rng_state, uint64_t l,
                     uint64_t row_begin, uint64_t row_end, uint32_t* mask_words) {
  API_TRY
  need_ctx(ctx);
  need_tensor(ctx);
  if (mode < 0 || mode >= ctx->order) fail(NTCB_ERANGE, "sample_mask: mode out of range");
  if (row_begin > row_end || row_end > ctx->dims[mode])
    fail(NTCB_ERANGE, "sample_mask: rows out of range");
  if (!(c > 0.0 && c < 1.0)) fail(NTCB_EINVAL, "sample_mask: c must be in (0, 1)");
  need_rows(ctx, mode, row_begin, row_end);
  collect(ctx, nullptr);
  const uint64_t* off = ctx->views[mode].h_off;
  const uint64_t e0 = off[row_begin], e1 = off[row_end];
  if (e1 <= e0) return NTCB_OK;
  host_of(ctx).prefetch[mode].valid = false;  // mask buffer 0 is overwritten below
  uint32_t* mask = ctx->mask[mode][0];
  const uint64_t w0 = e0 >> 5, w1 = ((e1 - 1) >> 5) + 1;
  NTCB_CUDA(cudaMemsetAsync(mask + w0, 0, sizeof(uint32_t) * (w1 - w0), ctx->stream));
  uint64_t cap = 0;
  const uint64_t root = fork64(rng_state, l);
  launch_sample_set(ctx, ctx->stream, mask, mode, row_begin, row_end, c, root, 0, &cap);
  launch_sample_heavy(ctx, ctx->stream, mask, mode, row_begin, row_end, c, root, 0, cap);
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
  NTCB_CUDA(cudaMemcpy(mask_words, mask + w0, sizeof(uint32_t) * (w1 - w0), cudaMemcpyDeviceToHost));
  API_CATCH
}

int ntcb_sweep_async(ntcb_context* ctx, uint64_t sweep, const ntcb_nmc_config* cfg, uint64_t seed) {
  API_TRY
  need_ctx(ctx);
  validate_nmc(cfg);
  need_factors(ctx);
  need_whole(ctx);
  for (int i = 0; i < ctx->order; ++i)
    if (!host_of(ctx).verified[i]) fail(NTCB_EINVAL, "s_nmc: a_init must be nonnegative");
  enqueue_sweep(ctx, sweep, *cfg, seed, false);
  API_CATCH
}

int ntcb_metrics(ntcb_context* ctx, double* sse, double* sumsq, double* reg) {
  API_TRY
  need_ctx(ctx);
  need_factors(ctx);
  collect(ctx, nullptr);
  double a, b, c;
  device_metrics(ctx, &a, &b, &c);
  if (sse) *sse = a;
  if (sumsq) *sumsq = b;
  if (reg) *reg = c;
  API_CATCH
}

int ntcb_objective(ntcb_context* ctx, double lambda, double* out) {
  API_TRY
  need_ctx(ctx);
  need_factors(ctx);
  if (lambda < 0.0) fail(NTCB_EINVAL, "objective: lambda must be >= 0");
  need_whole(ctx);
  double sse, sx, reg;
  device_metrics(ctx, &sse, &sx, &reg);
  *out = 0.5 * sse + 0.5 * lambda * reg;  // metrics.cpp:8-21
  API_CATCH
}

int ntcb_relative_error(ntcb_context* ctx, double* out) {
  API_TRY
  need_ctx(ctx);
  need_factors(ctx);
  need_whole(ctx);
  double sse, sx, reg;
  device_metrics(ctx, &sse, &sx, &reg);
  if (sx == 0.0) fail(NTCB_EDOMAIN, "relative_error: all observed values are zero");
  *out = std::sqrt(sse) / std::sqrt(sx);  // metrics.cpp:23-37
  API_CATCH
}

int ntcb_rmse(ntcb_context* ctx, double* out) {
  API_TRY
  need_ctx(ctx);
  need_factors(ctx);
  if (ctx->nnz == 0) fail(NTCB_EDOMAIN, "rmse: empty observation set");
  need_whole(ctx);
  double sse, sx, reg;
  device_metrics(ctx, &sse, &sx, &reg);
  *out = std::sqrt(sse / static_cast<double>(ctx->nnz));
  API_CATCH
}

int ntcb_ao_ntc(ntcb_context* ctx, const ntcb_ao_config* cfg, ntcb_metrics_record* history,
                uint64_t max_history, uint64_t* n_history, ntcb_observer_fn observer, void* user) {
  API_TRY
  need_ctx(ctx);
  if (!cfg) fail(NTCB_EINVAL, "AoConfig: null");
  // AoConfig::validate (ao.cpp:30-38)
  if (cfg->rank == 0) fail(NTCB_EINVAL, "AoConfig: rank must be positive");
  if (!(cfg->max_epochs >= 0.0)) fail(NTCB_EINVAL, "AoConfig: max_epochs must be >= 0");
  if (!(cfg->term_tol >= 0.0)) fail(NTCB_EINVAL, "AoConfig: term_tol must be >= 0");
  if (cfg->metrics_every < 1) fail(NTCB_EINVAL, "AoConfig: metrics_every must be >= 1");
  ntcb_nmc_config n{cfg->lambda, cfg->c, cfg->max_inner, cfg->power_iters, cfg->power_tol,
                    cfg->threads, cfg->chunk};
  validate_nmc(&n);
  need_factors(ctx);
  need_whole(ctx);
  if (ctx->rank != cfg->rank) fail(NTCB_EINVAL, "ao_ntc: init rank differs from configured rank");
  auto& hs = host_of(ctx);
  for (int m = 0; m < ctx->order; ++m)
    if (!hs.verified[m]) fail(NTCB_EINVAL, "ao_ntc: init factors must be nonnegative");
  collect(ctx, nullptr);

  // Device-resident loop (ao.cpp:75-133): the entries a sweep accesses are
  // known on the host before it runs (sum of floor(c n_p), nmc.cpp:36-40),
  // so the budget and zero-progress checks need no synchronisation; sweeps
  // are enqueued back to back and the host waits only where a record needs
  // device data (eval_metrics, an observer) and at the end.  Records without
  // device data take their wall_seconds from a CUDA event recorded after
  // their sweep (time since t0 at which the sweep finished on the device).
  std::vector<ntcb_metrics_record> hist;
  std::vector<std::pair<size_t, cudaEvent_t>> deferred;  // (record index, end-of-sweep event)
  struct EvFree {
    std::vector<std::pair<size_t, cudaEvent_t>>& d;
    cudaEvent_t base = nullptr;
    ~EvFree() {
      for (auto& x : d) cudaEventDestroy(x.second);
      if (base) cudaEventDestroy(base);
    }
  } evfree{deferred};
  uint64_t accessed = 0;
  const auto t0 = std::chrono::steady_clock::now();
  NTCB_CUDA(cudaEventCreate(&evfree.base));
  NTCB_CUDA(cudaEventRecord(evfree.base, ctx->stream));
  const double base_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const bool sync_records = cfg->eval_metrics || observer != nullptr;
  auto push = [&]() {
    ntcb_metrics_record r{};
    r.entries_accessed = accessed;
    if (ctx->nnz == 0) fail(NTCB_EINVAL, "epoch_fraction: empty observation set");
    r.epoch = static_cast<double>(accessed) / static_cast<double>(ctx->nnz);
    r.objective = std::nan("");
    r.rel_error = std::nan("");
    if (!sync_records) {
      cudaEvent_t e;
      NTCB_CUDA(cudaEventCreate(&e));
      NTCB_CUDA(cudaEventRecord(e, ctx->stream));
      deferred.emplace_back(hist.size(), e);
      hist.push_back(r);
      return;
    }
    collect(ctx, nullptr);  // queued sweeps done, first row failure reported
    r.wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (cfg->eval_metrics) {
      double sse, sx, reg;
      device_metrics(ctx, &sse, &sx, &reg);
      r.objective = 0.5 * sse + 0.5 * cfg->lambda * reg;
      if (sx == 0.0) fail(NTCB_EDOMAIN, "relative_error: all observed values are zero");
      r.rel_error = std::sqrt(sse) / std::sqrt(sx);
      if (!std::isfinite(r.objective)) fail(NTCB_ERUNTIME, "ao_ntc: objective diverged (non-finite)");
    }
    hist.push_back(r);
    if (observer) observer(&r, ctx, user);
  };
  push();
  bool last_recorded = true;
  for (uint64_t k = 0;; ++k) {
    if (static_cast<double>(accessed) / static_cast<double>(ctx->nnz) >= cfg->max_epochs) break;
    if (plateau(hist, cfg->term_tol)) break;
    const uint64_t st = enqueue_sweep(ctx, k, n, cfg->seed, true);
    if (st == 0) break;
    accessed += st;
    last_recorded = ((k + 1) % static_cast<uint64_t>(cfg->metrics_every) == 0);
    if (last_recorded) push();
  }
  if (!last_recorded) push();
  collect(ctx, nullptr);  // the remaining sweeps; a row failure throws here
  for (auto& x : deferred) {
    float ms = 0.f;
    NTCB_CUDA(cudaEventElapsedTime(&ms, evfree.base, x.second));
    hist[x.first].wall_seconds = base_s + 1e-3 * ms;
  }
  if (n_history) *n_history = hist.size();
  if (history)
    for (uint64_t i = 0; i < hist.size() && i < max_history; ++i) history[i] = hist[i];
  API_CATCH
}

int ntcb_render_model(ntcb_context* ctx, uint8_t* pixels) {
  API_TRY
  need_ctx(ctx);
  need_factors(ctx);
  if (ctx->order != 3 || ctx->dims[2] != 3)
    fail(NTCB_EINVAL, "render_model: expects an H x W x 3 factorization");  // image.cpp:162-163
  if (!pixels) fail(NTCB_EINVAL, "render_model: null pixels");
  collect(ctx, nullptr);
  const uint64_t n = 3 * ctx->dims[0] * ctx->dims[1];
  uint8_t* d = nullptr;
  NTCB_CUDA(cudaMalloc(&d, n ? n : 1));
  struct Free {
    uint8_t* p;
    ~Free() { cudaFree(p); }
  } fr{d};
  render_model(ctx, d);
  NTCB_CUDA(cudaMemcpyAsync(pixels, d, n, cudaMemcpyDeviceToHost, ctx->stream));
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_CATCH
}

int ntcb_profile_enable(ntcb_context* ctx, int on) {
  API_TRY
  need_ctx(ctx);
  ctx->prof.on = on != 0;
  ctx->prof.n = 0;
  ctx->prof.kn = 0;
  ctx->prof.launches = 0;
  ctx->prof.update_launches = 0;
  API_CATCH
}

int ntcb_profile_read(ntcb_context* ctx, double* update_ms, double* sample_ms, uint64_t* launches,
                      uint64_t* update_launches) {
  API_TRY
  need_ctx(ctx);
  NTCB_CUDA(cudaStreamSynchronize(ctx->side));
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
  Profile& pf = ctx->prof;
  double u = 0.0, s = 0.0;
  uint64_t nu = 0;
  for (int i = 0; i + 1 < pf.n; i += 2) {
    float ms = 0.f;
    NTCB_CUDA(cudaEventElapsedTime(&ms, pf.ev[i], pf.ev[i + 1]));
    if (pf.kind[i / 2] == 0) {
      u += ms;
      ++nu;
    } else {
      s += ms;
    }
  }
  if (update_ms) *update_ms = u;
  if (sample_ms) *sample_ms = s;
  if (launches) *launches = pf.launches;
  if (update_launches) *update_launches = nu;
  pf.n = 0;
  pf.launches = 0;
  pf.update_launches = 0;
  API_CATCH
}

int ntcb_profile_read_kernel(ntcb_context* ctx, double* item_kernel_ms, uint64_t* launches) {
  API_TRY
  need_ctx(ctx);
  NTCB_CUDA(cudaStreamSynchronize(ctx->stream));
  Profile& pf = ctx->prof;
  double t = 0.0;
  uint64_t n = 0;
  for (int i = 0; i + 1 < pf.kn; i += 2) {
    float ms = 0.f;
    NTCB_CUDA(cudaEventElapsedTime(&ms, pf.kev[i], pf.kev[i + 1]));
    t += ms;
    ++n;
  }
  if (item_kernel_ms) *item_kernel_ms = t;
  if (launches) *launches = n;
  pf.kn = 0;
  API_CATCH
}

}  // extern "C"
