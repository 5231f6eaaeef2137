/*
 * ntc_b200.h — C-ABI of the B200-native hot path of arXiv 2109.09534
 * (nonnegative tensor completion, per-mode stochastic accelerated projected
 * gradient "S_NMC" inside the AO sweep).
 *
 * The reference ("ntc", /root/reference/proj/core) is a C++20 library whose
 * hot path is called in-process; it has no FFI.  This header is the drop-in
 * boundary a C/C++/ctypes caller binds instead of the reference's C++ API.
 * Plain pointers and sizes only; no torch or CUDA types (streams cross as
 * void*).  Every entry point names the reference interface it replaces.
 *
 * Conventions
 *   - Return value: NTCB_OK (0) or an error code mirroring the C++ exception
 *     the reference throws in the same situation; ntcb_last_error() returns
 *     the message (same text as the reference's what()).
 *   - Host matrices are row-major double I x R, exactly ntc::Matrix
 *     (matrix.hpp:12-55).  On the device factors are fp32, row stride ld.
 *   - RNG streams cross as their raw 64-bit splitmix state: the state of
 *     ntc::RngStream (rng.hpp:13-63).  ntcb_sweep_stream_state() gives the
 *     state of sweep_stream(seed, k, mode) (ao.cpp:65-68).
 *   - Calls on one context are not re-entrant (like s_nmc, nmc.hpp:93-95).
 */
#ifndef NTC_B200_H_
#define NTC_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NTCB_OK 0
#define NTCB_EINVAL 1   /* std::invalid_argument */
#define NTCB_ERUNTIME 2 /* std::runtime_error    */
#define NTCB_ERANGE 3   /* std::out_of_range     */
#define NTCB_EDOMAIN 4  /* std::domain_error     */
#define NTCB_ECUDA 5    /* CUDA / device failure (no reference analogue) */

#define NTCB_MAX_ORDER 8
#define NTCB_MAX_RANK 64

typedef struct ntcb_context ntcb_context;

/* ntc::NmcConfig (nmc.hpp:13-23); validated like NmcConfig::validate
 * (nmc.cpp:13-23).  threads/chunk are validated and otherwise ignored: the
 * device schedule never changes results (nmc.hpp:89-92). */
typedef struct ntcb_nmc_config {
  double lambda;
  double c;
  int32_t max_inner;
  int32_t power_iters;
  double power_tol;
  int32_t threads;
  int32_t chunk;
} ntcb_nmc_config;

/* ntc::AoConfig (ao.hpp:12-29). */
typedef struct ntcb_ao_config {
  uint64_t rank;
  double lambda;
  double c;
  int32_t max_inner;
  int32_t power_iters;
  double max_epochs;
  double term_tol;
  uint64_t seed;
  int32_t threads;
  int32_t chunk;
  double power_tol;
  int32_t eval_metrics;
  int32_t metrics_every;
} ntcb_ao_config;

/* ntc::MetricsRecord (ao.hpp:31-37). */
typedef struct ntcb_metrics_record {
  double epoch;
  double objective;
  double rel_error;
  double wall_seconds;
  uint64_t entries_accessed;
} ntcb_metrics_record;

/* ntc::SweepObserver (ao.hpp:55): called after each record with the record;
 * factors are readable through ntcb_factor_get from inside the callback. */
typedef void (*ntcb_observer_fn)(const ntcb_metrics_record* rec, ntcb_context* ctx, void* user);

/* ---- library / context ------------------------------------------------- */
const char* ntcb_last_error(void);
int ntcb_version(void);
int ntcb_create(int device, ntcb_context** out);
int ntcb_destroy(ntcb_context* ctx);
/* Use the caller's cudaStream_t (e.g. torch.cuda.current_stream()); NULL
 * restores the context's own stream. */
int ntcb_set_stream(ntcb_context* ctx, void* cuda_stream);
int ntcb_synchronize(ntcb_context* ctx);
/* Page-locked host memory (cudaMallocHost) for factor buffers of the
 * host-buffer entry points; ntcb_host_free releases it. */
int ntcb_host_alloc(uint64_t bytes, void** out);
int ntcb_host_free(void* p);

/* ---- tuning (launch policy only; no reference analogue) -----------------
 * Per-context launch choices behind the measured defaults of DESIGN.md §3.
 * None of them changes results: every variant computes the same sampled
 * sets, and the update variants the same factors (they are A/B switches for
 * measurements, set through this struct -- never through the environment).
 * ntcb_tuning_defaults fills the defaults; ntcb_set_tuning validates and
 * applies (cached launch plans are rebuilt on demand). */
typedef struct ntcb_tuning {
  int32_t no_tc;             /* 1: CUDA-core Gram (k_update) instead of the tensor-core kernels */
  int32_t no_nat;            /* 1: ranks 25-32 without the natural-layout (NAT) gathers */
  int32_t tc_p;              /* 0 or 4: 4 = quad gather layout at ranks <= 31 (measured slower) */
  int32_t update_wpc;        /* warps per CTA of k_update_tc, 1..8 (default 4) */
  int64_t short_row;         /* average item length below which the SHORT update runs (2048) */
  int32_t side_sampler_ctas; /* CTAs per SM of the side-stream CTA sampler, 0 = no cap */
  int32_t heavy_per;         /* entries per thread when sizing heavy-slice sampler grids (8) */
  int32_t heavy_win_log2;    /* log2 of the heavy sampler's draw window (24) */
  int32_t heavy_big_log2;    /* log2 of the slice length taking the windowed path (24) */
  int32_t host_threads;      /* host threads for fp64 <-> fp32 factor conversion, 0 = min(cores, 16) */
  int32_t update_ctas_per_sm; /* resident update CTAs per SM (0 = as many as fit): fewer leave room
                                for the side-stream sampler of the next mode to run alongside */
  int32_t update_carveout;   /* shared-memory carve-out preference (percent) of the update kernels,
                                -1 = driver default; a smaller carve-out leaves more L1 for the
                                in-flight factor-row gathers at the cost of resident CTAs */
  int32_t graph;             /* 1: ntcb_sweep_async / ntcb_ao_ntc launch each sweep as one CUDA graph
                                (captured per sweep, updated in place), 0: stream launches */
  int32_t peer_fence;        /* ordering of the rows stored into peer replicas: 1 (default) one
                                system-scope fence per thread at kernel exit, 2 one per row,
                                0 none (the kernel boundary + the NCCL barrier alone) */
  int32_t nat_pad;           /* ranks 9-24, orders 3-4: whole-line factor rows + the natural-layout (NAT)
                                update -- 64-byte rows read by 4 lanes per pick up to rank 16, 128-byte
                                rows read by 8 lanes above (2: 128-byte rows at every rank, the A/B
                                reference); 1 on, 0 off, -1 (default) when the factors exceed 16 MB
                                (gathers mostly miss L1: configs 3 and 5 measured 2.6 % / 5 % faster,
                                configs 1 and 2, whose factors stay cached, slower) */
  int32_t tiny_sampler;      /* 1 (default): slices of at most 64 entries are sampled by one lane each
                                (k_sample_tiny) when a mode has thousands of them; 0: a warp per slice */
  int32_t item_order;        /* work-list order of equally long update items: 0 row-major (a row's chunks
                                together), 1 chunk-major (chunk s of every row together: co-resident
                                warps gather the same window of the slowest-varying other factor, so
                                its rows hit L1) */
} ntcb_tuning;
void ntcb_tuning_defaults(ntcb_tuning* t);
int ntcb_set_tuning(ntcb_context* ctx, const ntcb_tuning* t);
int ntcb_get_tuning(ntcb_context* ctx, ntcb_tuning* t);

/* ---- RNG (rng.hpp:13-63, ao.cpp:65-68) — host-side helpers ------------- */
uint64_t ntcb_rng_fork(uint64_t state, uint64_t tag);
uint64_t ntcb_sweep_stream_state(uint64_t seed, uint64_t sweep, int mode);

/* ---- tensor + mode views ------------------------------------------------
 * Replaces ntc::SparseTensor(dims, indices, values) (sparse_tensor.cpp:24-73)
 * followed by build_mode_views (mode_view.cpp:8-37).  indices: nnz*order
 * 0-based coordinates, entry-major, any order; values: double (rounded to
 * fp32 on the device, the path's arithmetic type).  Validation, canonical
 * lexicographic sort, duplicate detection and the per-mode stable views are
 * all built on the device; same error texts as the reference. */
int ntcb_tensor_load(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                     const uint32_t* indices, const double* values);
/* Same, with fp32 values (the benchmark path: no double staging). */
int ntcb_tensor_load_f32(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                         const uint32_t* indices, const float* values);
/* Same, inputs already in device memory (e.g. from ntcb_synth_*). */
int ntcb_tensor_load_device(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                            const uint32_t* d_indices, const float* d_values);
int ntcb_tensor_info(ntcb_context* ctx, int* order, uint64_t* dims, uint64_t* nnz);
/* ModeView export (mode_view.hpp:13-29): offsets[dims[mode]+1],
 * others[nnz*(order-1)], values[nnz]; any pointer may be NULL. */
int ntcb_view_export(ntcb_context* ctx, int mode, uint64_t* offsets, uint32_t* others,
                     float* values);
/* Rows [row_begin, row_end) of a view: offsets[row_end-row_begin+1]
 * (absolute entry positions), others/values of those slices only. */
int ntcb_view_export_rows(ntcb_context* ctx, int mode, uint64_t row_begin, uint64_t row_end,
                          uint64_t* offsets, uint32_t* others, float* values);
/* Slab storage for row-sharded multi-GPU runs: keep only the entries of
 * rows [row_begin, row_end) of view `mode` on the device (within the rows
 * already kept), freeing the rest -- every rank of an N-way run then holds
 * ~1/N of each view.  Afterwards only calls on those rows are accepted
 * (ntcb_s_nmc_rows_async, ntcb_sample_rows / _row / _mask, the row export);
 * whole-mode calls fail with NTCB_ERANGE, and ntcb_metrics returns the
 * partial sums over the kept rows of mode 0 (sum them over the ranks).
 * ntcb_view_resident reports the kept rows and the device bytes of the view. */
int ntcb_view_keep_rows(ntcb_context* ctx, int mode, uint64_t row_begin, uint64_t row_end);
int ntcb_view_resident(ntcb_context* ctx, int mode, uint64_t* row_begin, uint64_t* row_end,
                       uint64_t* device_bytes);
/* Canonical (lexicographic) COO, SparseTensor::indices()/values(). */
int ntcb_tensor_export(ntcb_context* ctx, uint32_t* indices, float* values);

/* ---- .tns files (tns_io.cpp:41-142), parallel host parser --------------
 * Same syntax and diagnostics as read_tns ("path:line: message",
 * std::runtime_error -> NTCB_ERUNTIME).  ntcb_tns_parse allocates *indices
 * (nnz*order, 0-based) and *values with malloc (release with ntcb_free);
 * host only, no device needed; its message is in ntcb_tns_last_error().
 * ntcb_tensor_read_tns parses and loads (validation, canonical order and
 * views on the device); ntcb_tns_write writes "# dims:" + 1-based %.17g. */
int ntcb_tns_parse(const char* path, int* order, uint64_t* dims, uint64_t* nnz,
                   uint32_t** indices, double** values);
const char* ntcb_tns_last_error(void);
void ntcb_free(void* p);
int ntcb_tns_write(const char* path, int order, const uint64_t* dims, uint64_t nnz,
                   const uint32_t* indices, const double* values);
int ntcb_tensor_read_tns(ntcb_context* ctx, const char* path);

/* ---- factors (FactorSet, factor_set.hpp:12-35) ------------------------- */
/* factors/momentum: order pointers to host row-major double dims[m] x rank;
 * momentum may be NULL (= factors).  Factors must be nonnegative. */
int ntcb_factors_init(ntcb_context* ctx, uint64_t rank, const double* const* factors,
                      const double* const* momentum);
/* initial_factors(dims, rank, seed) (ao.cpp:70-73) generated on the device. */
int ntcb_factors_random(ntcb_context* ctx, uint64_t rank, uint64_t seed);
int ntcb_factor_set(ntcb_context* ctx, int mode, const double* a, const double* y);
int ntcb_factor_get(ntcb_context* ctx, int mode, double* a, double* y);
/* Device pointers of factor A (which=0) or momentum Y (which=1): fp32,
 * dims[mode] rows, row stride *ld floats (ld >= rank, padding is zero). */
int ntcb_factor_device_ptr(ntcb_context* ctx, int mode, int which, void** ptr, uint64_t* ld);

/* ---- fused exchange for row-sharded multi-GPU runs -----------------------
 * Replicas of factor A[mode] on other GPUs (same dims, same ld) can be
 * registered as peers: every row an S_NMC call finalises is then also
 * stored into each peer replica by the update kernel itself (NVLink P2P
 * stores, issued row by row while other rows are still computing), so a
 * row-sharded sweep needs only a barrier after each mode instead of an
 * all-gather.  The peers see the rows once this call's kernels completed
 * and a cross-GPU barrier ordered after them (e.g. a one-element NCCL
 * all-reduce on the library stream) returned.
 * ntcb_factor_ipc_handle: the CUDA IPC handle (64 bytes) of A[mode];
 * ntcb_ipc_open: maps another process's handle into this one (lazy peer
 * access); ntcb_factor_set_peers: registers n <= 7 device pointers to peer
 * replicas of A[mode] (n = 0 clears). */
int ntcb_factor_ipc_handle(ntcb_context* ctx, int mode, void* handle64);
int ntcb_ipc_open(ntcb_context* ctx, const void* handle64, void** ptr);
int ntcb_factor_set_peers(ntcb_context* ctx, int mode, int n, void* const* peer_ptrs);

/* ---- S_NMC (nmc.hpp:93-95, nmc.cpp:199-272) -----------------------------
 * One call = one ntc::s_nmc(views[mode], factors, mode, a_init, cfg,
 * RngStream(rng_state), &stats): A = Y = a_init, then max_inner inner
 * iterations over every row (sample, gradient at Y, Hessian, 1.01 x power
 * method, projected Nesterov step).  a_init == NULL aliases factors[mode]
 * (as ao_ntc does, ao.cpp:123); otherwise a host double dims[mode] x rank.
 * *entries_accessed is ADDED to (nmc.cpp:270); may be NULL. */
int ntcb_s_nmc(ntcb_context* ctx, int mode, const double* a_init, const ntcb_nmc_config* cfg,
               uint64_t rng_state, uint64_t* entries_accessed);
/* Host-buffer drop-in: a_init in, updated factors[mode] (a_out) and
 * momentum[mode] (y_out) out, all host double; H2D/D2H inside the call.
 * When every buffer is page-locked (e.g. from ntcb_host_alloc) the fp64 <->
 * fp32 conversion and the nonnegativity check run on the device and the
 * copies go straight to and from the caller's arrays; otherwise the call
 * converts on the host through its own pinned staging.  Same results. */
int ntcb_s_nmc_host(ntcb_context* ctx, int mode, const double* a_init, double* a_out,
                    double* y_out, const ntcb_nmc_config* cfg, uint64_t rng_state,
                    uint64_t* entries_accessed);
/* Optional hint for drivers built on ntcb_s_nmc / ntcb_s_nmc_host: the
 * sampled set of a FUTURE call's first inner iteration (same mode, cfg->c
 * and rng_state) is drawn now, on the sampler stream, while earlier work
 * runs -- the sets depend on the stream state only (nmc.cpp:44-63), never
 * on the factors, and ao_ntc's states are known ahead (sweep_stream,
 * ao.cpp:65-68).  The matching call consumes it; any other sampling of the
 * mode in between discards it.  Results are identical with or without. */
int ntcb_sample_prefetch(ntcb_context* ctx, int mode, const ntcb_nmc_config* cfg, uint64_t rng_state);
/* Row shard [row_begin, row_end) of the same update (multi-GPU partition;
 * rows are independent, nmc.cpp:231).  a_init aliases factors[mode].
 * Asynchronous: errors and the count are collected by ntcb_collect(). */
int ntcb_s_nmc_rows_async(ntcb_context* ctx, int mode, uint64_t row_begin, uint64_t row_end,
                          const ntcb_nmc_config* cfg, uint64_t rng_state);
/* Heavy rows shared by several ranks (max_inner = 1).  A row of a mode is cut
 * into ntcb_segment_length()-entry chunks from its start (a property of the
 * mode: any partition cuts it the same way).  ntcb_s_nmc_chunks_async samples
 * the row (its stream RngStream(rng_state).fork(0).fork(row)) and writes the
 * fp32 (H, w) partials of chunks [chunk_begin, chunk_end) -- R*R + R floats
 * each, in chunk order -- to the device buffer d_slots, finalising nothing;
 * ntcb_finalize_row_async takes the row's complete set (every chunk, in
 * order, gathered from the ranks) and sums, steps and stores the row exactly
 * as a single-GPU call does (bitwise), counting its entries once. */
int ntcb_segment_length(ntcb_context* ctx, int mode, uint64_t* seg);
int ntcb_s_nmc_chunks_async(ntcb_context* ctx, int mode, uint64_t row, uint32_t chunk_begin,
                            uint32_t chunk_end, const ntcb_nmc_config* cfg, uint64_t rng_state,
                            void* d_slots);
int ntcb_finalize_row_async(ntcb_context* ctx, int mode, uint64_t row, const void* d_slots,
                            uint32_t nslots, const ntcb_nmc_config* cfg);
/* Waits for queued work; adds the entries accessed since the last collect
 * to *entries_accessed and reports the first row failure (lowest row). */
int ntcb_collect(ntcb_context* ctx, uint64_t* entries_accessed);

/* sample_row for every row in [row_begin, row_end) of view `mode` with the
 * row stream RngStream(rng_state).fork(l).fork(p) (nmc.cpp:236): writes
 * pick_offsets[row_end-row_begin+1] and the picks (slice-local offsets, in
 * draw order, nmc.cpp:44-63) to host buffers; picks may be NULL to query
 * the total (pick_offsets[last]). */
int ntcb_sample_rows(ntcb_context* ctx, int mode, double c, uint64_t rng_state, uint64_t l,
                     uint64_t row_begin, uint64_t row_end, uint64_t* pick_offsets,
                     uint32_t* picks);

/* The production sampled-set path used by the update (mask of the picks of
 * every row in [row_begin, row_end) for the row streams
 * RngStream(rng_state).fork(l).fork(p)): copies the mask words covering the
 * rows' entries, word (off[row_begin] >> 5) first, into mask_words. */
int ntcb_sample_mask(ntcb_context* ctx, int mode, double c, uint64_t rng_state, uint64_t l,
                     uint64_t row_begin, uint64_t row_end, uint32_t* mask_words);
/* ntc::sample_row(view, row, c, RngStream(row_state)) (nmc.hpp:45,
 * nmc.cpp:110-118): one row, the stream used as is.  *count receives
 * floor(c * n); picks (capacity >= slice length) may be NULL to query. */
int ntcb_sample_row(ntcb_context* ctx, int mode, uint64_t row, double c, uint64_t row_state,
                    uint32_t* picks, uint64_t* count);

/* ---- AO driver (ao.cpp:75-133) ----------------------------------------- */
/* One AO iteration k: s_nmc for modes 0..N-1 with sweep_stream(seed,k,i)
 * (Gauss-Seidel, ao.cpp:121-124).  Asynchronous; see ntcb_collect. */
int ntcb_sweep_async(ntcb_context* ctx, uint64_t sweep, const ntcb_nmc_config* cfg,
                     uint64_t seed);
/* ao_ntc on the resident tensor and factors (factors are the init). */
int ntcb_ao_ntc(ntcb_context* ctx, const ntcb_ao_config* cfg, ntcb_metrics_record* history,
                uint64_t max_history, uint64_t* n_history, ntcb_observer_fn observer,
                void* user);

/* ---- metrics (metrics.cpp:8-37) ---------------------------------------- */
/* sse = sum_Omega (x - model)^2, sumsq = sum x^2, reg = sum_m ||U_m||_F^2
 * (sse and sumsq over the kept rows of mode 0 when the view is a slab). */
int ntcb_metrics(ntcb_context* ctx, double* sse, double* sumsq, double* reg);
int ntcb_objective(ntcb_context* ctx, double lambda, double* out);
int ntcb_relative_error(ntcb_context* ctx, double* out);
/* masked RMSE = sqrt(sse / |Omega|). */
int ntcb_rmse(ntcb_context* ctx, double* out);

/* ---- image demo (image.cpp:161-183) ------------------------------------ */
/* render_model: the dense H x W x 3 evaluation of the resident factors
 * (order 3, dims[2] == 3) into 8-bit pixels, row-major (i, j, channel),
 * quantize = lround(clamp(v, 0, 255)); fp64 sums on the device.  pixels:
 * host buffer of 3 * dims[0] * dims[1] bytes.  invalid_argument (same text
 * as the reference) for any other shape. */
int ntcb_render_model(ntcb_context* ctx, uint8_t* pixels);

/* ---- synthetic data (BASELINE.json configs; not in the reference) ------ */
/* Uniform unique cells + rank-`true_rank` U[0,1) CPD values + N(0,sigma^2)
 * noise clamped at 0, generated on the device from `seed`; writes device
 * buffers owned by the context, then loads them as the tensor. */
int ntcb_synth_uniform(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
                       uint64_t true_rank, double sigma, uint64_t seed);

/* General form: zipf_alpha[m] > 0 draws mode m from Zipf(alpha) over a
 * seeded permutation of the ids (NULL or 0 = uniform); value_kind 0 = CPD +
 * noise clamped at 0, 1 = round(clip(1 + 4 CPD/true_rank + noise, 1, 5)). */
int ntcb_synth(ntcb_context* ctx, int order, const uint64_t* dims, uint64_t nnz,
               uint64_t true_rank, double sigma, uint64_t seed, const double* zipf_alpha,
               int value_kind);

/* ---- timing hooks for bench.py ----------------------------------------- */
/* Kernel-level timing since profiling was enabled (or the last read): total
 * device ms of the timed mode updates (update kernel + split-row
 * finalisation, CUDA events on the context stream) and of the sampler phases
 * (side stream), the number of kernel launches issued, and the number of
 * timed mode updates (update_launches; at most 2048 phases are timed). */
int ntcb_profile_enable(ntcb_context* ctx, int on);
/* The update's item kernel alone (gradient + Hessian + row end of unsplit rows; without the
 * split-row finalisation kernels): summed device time and launch count since profiling was
 * enabled or last read. */
int ntcb_profile_read_kernel(ntcb_context* ctx, double* item_kernel_ms, uint64_t* launches);
int ntcb_profile_read(ntcb_context* ctx, double* update_ms, double* sample_ms,
                      uint64_t* launches, uint64_t* update_launches);

#ifdef __cplusplus
}
#endif

#endif /* NTC_B200_H_ */
