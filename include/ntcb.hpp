// ntcb.hpp — C++ host API over the C-ABI (ntc_b200.h), mirroring the names,
// argument meaning and exceptions of the reference's proj/core API for the
// hot path (ntc::RngStream, NmcConfig, AoConfig, MetricsRecord, s_nmc,
// ao_ntc, objective, relative_error, sweep_stream, initial_factors).
// Header-only; link with libntcb.so.  A reference user swaps
//   #include "ntc/ao.hpp"            ->  #include "ntcb.hpp"
//   ntc::s_nmc(views[i], f, i, ...)  ->  solver.s_nmc(i, a_init, cfg, rng, &stats)
// (see INTEGRATION.md).  Factors live on the device between calls; host
// matrices are row-major double I x R like ntc::Matrix (matrix.hpp:12-55).
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "ntc_b200.h"

namespace ntcb {

[[noreturn]] inline void throw_code(int rc) {
  const std::string msg = ntcb_last_error();
  switch (rc) {
    case NTCB_EINVAL: throw std::invalid_argument(msg);
    case NTCB_ERANGE: throw std::out_of_range(msg);
    case NTCB_EDOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);  // NTCB_ERUNTIME, NTCB_ECUDA
  }
}
inline void check(int rc) {
  if (rc != NTCB_OK) throw_code(rc);
}

// ntc::RngStream (rng.hpp:13-63) plus the raw state accessor the C-ABI needs.
class RngStream {
 public:
  explicit RngStream(std::uint64_t seed) : state_(seed) {}
  RngStream fork(std::uint64_t tag) const { return RngStream(ntcb_rng_fork(state_, tag)); }
  std::uint64_t state() const { return state_; }

 private:
  std::uint64_t state_;
};

// ntc::sweep_stream (ao.cpp:65-68)
inline RngStream sweep_stream(std::uint64_t seed, std::uint64_t sweep, int mode) {
  return RngStream(ntcb_sweep_stream_state(seed, sweep, mode));
}

// ntc::NmcConfig (nmc.hpp:13-23)
struct NmcConfig {
  double lambda = 1e-3;
  double c = 1.0;
  int max_inner = 1;
  int power_iters = 30;
  double power_tol = 1e-6;
  int threads = 1;
  int chunk = 0;
  ntcb_nmc_config c_config() const {
    return ntcb_nmc_config{lambda, c, max_inner, power_iters, power_tol, threads, chunk};
  }
};

// ntc::AoConfig (ao.hpp:12-29)
struct AoConfig {
  std::size_t rank = 1;
  double lambda = 1e-3;
  double c = 1.0;
  int max_inner = 1;
  double max_epochs = 100.0;
  double term_tol = 0.0;
  std::uint64_t seed = 0;
  int threads = 1;
  int chunk = 0;
  int power_iters = 30;
  double power_tol = 1e-6;
  bool eval_metrics = true;
  int metrics_every = 1;
  NmcConfig nmc() const {
    NmcConfig n;
    n.lambda = lambda;
    n.c = c;
    n.max_inner = max_inner;
    n.power_iters = power_iters;
    n.power_tol = power_tol;
    n.threads = threads;
    n.chunk = chunk;
    return n;
  }
};

using MetricsRecord = ntcb_metrics_record;  // ntc::MetricsRecord (ao.hpp:31-37)

struct SnmcStats {  // ntc::SnmcStats (nmc.hpp:73-75)
  std::uint64_t entries_accessed = 0;
};

// A device context holding the tensor's mode views and the FactorSet.
class Solver {
 public:
  explicit Solver(int device = 0) { check(ntcb_create(device, &ctx_)); }
  ~Solver() { ntcb_destroy(ctx_); }
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  // ntc::SparseTensor(dims, indices, values) + build_mode_views.
  void load(const std::vector<std::size_t>& dims, const std::vector<std::uint32_t>& indices,
            const std::vector<double>& values) {
    std::vector<std::uint64_t> d(dims.begin(), dims.end());
    if (dims.size() >= 2 && indices.size() != values.size() * dims.size())
      throw std::invalid_argument("SparseTensor: index/value length mismatch");
    check(ntcb_tensor_load(ctx_, static_cast<int>(d.size()), d.data(), values.size(),
                           indices.data(), values.data()));
    dims_ = dims;
  }

  // FactorSet (factor_set.hpp:12-35): factors[m] is dims[m] x rank row-major.
  void set_factors(std::size_t rank, const std::vector<std::vector<double>>& factors) {
    std::vector<const double*> p;
    for (const auto& f : factors) p.push_back(f.data());
    check(ntcb_factors_init(ctx_, rank, p.data(), nullptr));
    rank_ = rank;
  }
  // initial_factors(dims, rank, seed) (ao.cpp:70-73), generated on the device.
  void initial_factors(std::size_t rank, std::uint64_t seed) {
    check(ntcb_factors_random(ctx_, rank, seed));
    rank_ = rank;
  }
  std::vector<double> factor(int mode) const {
    std::vector<double> a(dims_.at(mode) * rank_);
    check(ntcb_factor_get(ctx_, mode, a.data(), nullptr));
    return a;
  }
  std::vector<double> momentum(int mode) const {
    std::vector<double> y(dims_.at(mode) * rank_);
    check(ntcb_factor_get(ctx_, mode, nullptr, y.data()));
    return y;
  }

  // ntc::s_nmc (nmc.hpp:93-95).  a_init == nullptr aliases factors[mode]
  // (as ao_ntc passes it, ao.cpp:123); returns the updated factor.
  std::vector<double> s_nmc(int mode, const std::vector<double>* a_init, const NmcConfig& cfg,
                            RngStream rng, SnmcStats* stats = nullptr) {
    const ntcb_nmc_config c = cfg.c_config();
    std::uint64_t acc = 0;
    check(ntcb_s_nmc(ctx_, mode, a_init ? a_init->data() : nullptr, &c, rng.state(), &acc));
    if (stats) stats->entries_accessed += acc;
    return factor(mode);
  }

  // Optional hint: draw the first sampled set of a later s_nmc(mode, ..., cfg, rng)
  // now, while earlier work runs (ntcb_sample_prefetch); results are unchanged.
  void sample_prefetch(int mode, const NmcConfig& cfg, RngStream rng) {
    const ntcb_nmc_config c = cfg.c_config();
    check(ntcb_sample_prefetch(ctx_, mode, &c, rng.state()));
  }

  // ntc::ao_ntc (ao.cpp:75-133) on the loaded tensor; the factors are the init.
  std::vector<MetricsRecord> ao_ntc(const AoConfig& cfg,
                                    const std::function<void(const MetricsRecord&)>& obs = {}) {
    ntcb_ao_config c{cfg.rank,      cfg.lambda,         cfg.c,          cfg.max_inner,
                     cfg.power_iters, cfg.max_epochs,    cfg.term_tol,   cfg.seed,
                     cfg.threads,   cfg.chunk,           cfg.power_tol,  cfg.eval_metrics ? 1 : 0,
                     cfg.metrics_every};
    std::vector<MetricsRecord> hist(1 << 16);
    std::uint64_t n = 0;
    auto tramp = [](const ntcb_metrics_record* r, ntcb_context*, void* user) {
      (*static_cast<const std::function<void(const MetricsRecord&)>*>(user))(*r);
    };
    check(ntcb_ao_ntc(ctx_, &c, hist.data(), hist.size(), &n, obs ? +tramp : nullptr,
                      obs ? const_cast<void*>(static_cast<const void*>(&obs)) : nullptr));
    hist.resize(n);
    return hist;
  }

  double objective(double lambda) const {  // metrics.cpp:8-21
    double out = 0;
    check(ntcb_objective(ctx_, lambda, &out));
    return out;
  }
  double relative_error() const {  // metrics.cpp:23-37
    double out = 0;
    check(ntcb_relative_error(ctx_, &out));
    return out;
  }
  // render_model (image.cpp:161-183): H x W x 3 pixels, row-major
  std::vector<std::uint8_t> render_model() const {
    std::vector<std::uint8_t> px(3 * (dims_.size() >= 2 ? dims_[0] * dims_[1] : 0));
    check(ntcb_render_model(ctx_, px.data()));
    return px;
  }
  // slab storage for a row shard (multi-GPU): only rows [r0, r1) of view `mode` stay resident
  void keep_rows(int mode, std::uint64_t r0, std::uint64_t r1) { check(ntcb_view_keep_rows(ctx_, mode, r0, r1)); }
  // launch policy (never changes results)
  ntcb_tuning tuning() const {
    ntcb_tuning t;
    check(ntcb_get_tuning(ctx_, &t));
    return t;
  }
  void set_tuning(const ntcb_tuning& t) { check(ntcb_set_tuning(ctx_, &t)); }
  ntcb_context* handle() const { return ctx_; }

 private:
  ntcb_context* ctx_ = nullptr;
  std::vector<std::size_t> dims_;
  std::size_t rank_ = 0;
};

}  // namespace ntcb
