// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library ntc::core, compiled
// from the sources under /root/reference/proj/core by oracle/Makefile into
// oracle/_ref/libntc_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline leg / --impl reference) load it, as the checker or
// as the timed reference arm.  Nothing here re-implements the algorithm: every
// numeric result comes from the reference's own functions:
//   RngStream            proj/core/include/ntc/rng.hpp:13-63
//   SparseTensor ctor    proj/core/src/sparse_tensor.cpp:24-73
//   build_mode_views     proj/core/src/mode_view.cpp:8-37
//   sample_row           proj/core/src/nmc.cpp:110-118
//   row_gradient/hessian proj/core/src/nmc.cpp:120-138
//   power_method         proj/core/src/nmc.cpp:140-172
//   row_step             proj/core/src/nmc.cpp:174-197
//   s_nmc                proj/core/src/nmc.cpp:199-272
//   objective/rel_error  proj/core/src/metrics.cpp:8-37
//   render_model         proj/core/src/image.cpp:161-183
//   ao_ntc/sweep_stream  proj/core/src/ao.cpp:65-133
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "ntc/ao.hpp"
#include "ntc/factor_set.hpp"
#include "ntc/image.hpp"
#include "ntc/metrics.hpp"
#include "ntc/mode_view.hpp"
#include "ntc/nmc.hpp"
#include "ntc/rng.hpp"
#include "ntc/sparse_tensor.hpp"
#include "ntc/tns_io.hpp"

namespace {

thread_local std::string g_err;

// Error codes mirror the exception type so the Python side can re-raise the
// same class: 1 invalid_argument, 2 runtime_error, 3 out_of_range,
// 4 domain_error, 5 other.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 3;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

struct Problem {
  std::vector<std::size_t> dims;
  std::optional<ntc::SparseTensor> tensor;
  std::vector<ntc::ModeView> views;
  std::optional<ntc::FactorSet> factors;
};

ntc::Matrix to_matrix(const double* p, std::size_t rows, std::size_t cols) {
  ntc::Matrix m(rows, cols);
  if (rows * cols) std::memcpy(m.data().data(), p, sizeof(double) * rows * cols);
  return m;
}

}  // namespace

extern "C" {

struct ref_nmc_cfg {
  double lambda;
  double c;
  int max_inner;
  int power_iters;
  double power_tol;
  int threads;
  int chunk;
};

struct ref_ao_cfg {
  std::uint64_t rank;
  double lambda;
  double c;
  int max_inner;
  double max_epochs;
  double term_tol;
  std::uint64_t seed;
  int threads;
  int chunk;
  int power_iters;
  double power_tol;
  int eval_metrics;
  int metrics_every;
};

const char* ref_last_error() { return g_err.c_str(); }

// ---- RNG (rng.hpp) --------------------------------------------------------
int ref_rng_next_u64(std::uint64_t state, int n, std::uint64_t* out) {
  ntc::RngStream s(state);
  for (int i = 0; i < n; ++i) out[i] = s.next_u64();
  return 0;
}
int ref_rng_next_double(std::uint64_t state, int n, double* out) {
  ntc::RngStream s(state);
  for (int i = 0; i < n; ++i) out[i] = s.next_double();
  return 0;
}
int ref_rng_next_below(std::uint64_t state, std::uint64_t bound, int n, std::uint64_t* out) {
  ntc::RngStream s(state);
  for (int i = 0; i < n; ++i) out[i] = s.next_below(bound);
  return 0;
}
// First draw of RngStream(state).fork(tag) — pins fork() without the private state.
std::uint64_t ref_rng_fork_first(std::uint64_t state, std::uint64_t tag) {
  return ntc::RngStream(state).fork(tag).next_u64();
}
// First draw of sweep_stream(seed, k, mode).fork(l).fork(p) (ao.cpp:65-68, nmc.cpp:236).
std::uint64_t ref_row_stream_first(std::uint64_t seed, std::uint64_t k, int mode,
                                   std::uint64_t l, std::uint64_t p) {
  return ntc::sweep_stream(seed, k, mode).fork(l).fork(p).next_u64();
}
std::uint64_t ref_mix(std::uint64_t z) { return ntc::RngStream::mix(z); }

// ---- problem handle -------------------------------------------------------
void* ref_tensor_new(int order, const std::uint64_t* dims, std::uint64_t nnz,
                     const std::uint32_t* idx, const double* vals) {
  Problem* out = nullptr;
  int rc = guarded([&] {
    auto p = std::make_unique<Problem>();
    p->dims.assign(dims, dims + order);
    std::vector<ntc::coord_t> ix(idx, idx + nnz * static_cast<std::uint64_t>(order));
    std::vector<double> vs(vals, vals + nnz);
    p->tensor.emplace(p->dims, std::move(ix), std::move(vs));
    p->views = ntc::build_mode_views(*p->tensor);
    out = p.release();
  });
  return rc == 0 ? out : nullptr;
}

// Views filled directly (bounded CPU-baseline samples): view m holds
// view_rows[m] slices with the given CSR arrays; no SparseTensor exists, so
// metrics/ao entry points reject this handle.
void* ref_views_new(int order, const std::uint64_t* dims, const std::uint64_t* view_rows,
                    const std::uint64_t* const* offsets, const std::uint32_t* const* others,
                    const double* const* values) {
  Problem* out = nullptr;
  int rc = guarded([&] {
    auto p = std::make_unique<Problem>();
    p->dims.assign(dims, dims + order);
    p->views.resize(order);
    for (int m = 0; m < order; ++m) {
      ntc::ModeView& v = p->views[m];
      v.mode = m;
      v.order = order;
      const std::uint64_t rows = view_rows[m];
      v.offsets.assign(offsets[m], offsets[m] + rows + 1);
      const std::uint64_t base = v.offsets[0];
      for (auto& o : v.offsets) o -= base;
      const std::uint64_t n = v.offsets.back();
      v.values.assign(values[m] + base, values[m] + base + n);
      v.others.assign(others[m] + base * (order - 1), others[m] + (base + n) * (order - 1));
    }
    out = p.release();
  });
  return rc == 0 ? out : nullptr;
}

void ref_free(void* h) { delete static_cast<Problem*>(h); }

std::uint64_t ref_nnz(void* h) {
  auto* p = static_cast<Problem*>(h);
  return p->tensor ? p->tensor->nnz() : 0;
}

int ref_tensor_export(void* h, std::uint32_t* idx, double* vals) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    if (!p->tensor) throw std::invalid_argument("ref_tensor_export: no tensor");
    auto ix = p->tensor->indices();
    auto vs = p->tensor->values();
    std::copy(ix.begin(), ix.end(), idx);
    std::copy(vs.begin(), vs.end(), vals);
  });
}

std::uint64_t ref_view_rows(void* h, int mode) {
  return static_cast<Problem*>(h)->views[mode].slice_count();
}
std::uint64_t ref_view_nnz(void* h, int mode) {
  return static_cast<Problem*>(h)->views[mode].offsets.back();
}

int ref_view_export(void* h, int mode, std::uint64_t* offsets, std::uint32_t* others,
                    double* values) {
  return guarded([&] {
    const auto& v = static_cast<Problem*>(h)->views.at(mode);
    std::copy(v.offsets.begin(), v.offsets.end(), offsets);
    std::copy(v.others.begin(), v.others.end(), others);
    std::copy(v.values.begin(), v.values.end(), values);
  });
}

int ref_sample_row(void* h, int mode, std::uint64_t row, double c, std::uint64_t state,
                   std::uint32_t* picks, std::uint64_t* count) {
  return guarded([&] {
    const auto& v = static_cast<Problem*>(h)->views.at(mode);
    ntc::SampledRow s = ntc::sample_row(v, row, c, ntc::RngStream(state));
    std::copy(s.picks.begin(), s.picks.end(), picks);
    *count = s.picks.size();
  });
}

int ref_factors_init(void* h, std::uint64_t rank, const double* const* fac,
                     const double* const* mom) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    ntc::FactorSet f = ntc::FactorSet::zeros(p->dims, rank);
    for (std::size_t m = 0; m < p->dims.size(); ++m) {
      f.factors[m] = to_matrix(fac[m], p->dims[m], rank);
      f.momentum[m] = to_matrix(mom ? mom[m] : fac[m], p->dims[m], rank);
    }
    p->factors.emplace(std::move(f));
  });
}

// Replace the rows of factor `mode` (used by the bounded sample, whose
// factors[mode] has only the sampled rows).
int ref_factor_resize(void* h, int mode, std::uint64_t rows, const double* a) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    if (!p->factors) throw std::invalid_argument("ref_factor_resize: no factors");
    p->factors->factors.at(mode) = to_matrix(a, rows, p->factors->rank);
    p->factors->momentum.at(mode) = p->factors->factors[mode];
  });
}

int ref_factors_get(void* h, int mode, double* a, double* y) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    if (!p->factors) throw std::invalid_argument("ref_factors_get: no factors");
    const auto& A = p->factors->factors.at(mode);
    const auto& Y = p->factors->momentum.at(mode);
    if (a) std::copy(A.data().begin(), A.data().end(), a);
    if (y) std::copy(Y.data().begin(), Y.data().end(), y);
  });
}

// s_nmc on view `mode`.  a_init == NULL aliases factors[mode] exactly as
// ao_ntc does (ao.cpp:122-124); the stream is RngStream(rng_state).
int ref_s_nmc(void* h, int mode, const double* a_init, std::uint64_t a_rows,
              const ref_nmc_cfg* cfg, std::uint64_t rng_state, std::uint64_t* accessed) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    if (!p->factors) throw std::invalid_argument("ref_s_nmc: no factors");
    ntc::NmcConfig c;
    c.lambda = cfg->lambda;
    c.c = cfg->c;
    c.max_inner = cfg->max_inner;
    c.power_iters = cfg->power_iters;
    c.power_tol = cfg->power_tol;
    c.threads = cfg->threads;
    c.chunk = cfg->chunk;
    ntc::SnmcStats st;
    if (mode < 0 || static_cast<std::size_t>(mode) >= p->views.size()) {
      // let the reference produce its own diagnostic for a bad mode
      ntc::s_nmc(p->views.at(0), *p->factors, mode, p->factors->factors.at(0), c,
                 ntc::RngStream(rng_state), &st);
    }
    if (a_init) {
      const ntc::Matrix ai = to_matrix(a_init, a_rows, p->factors->rank);
      ntc::s_nmc(p->views[mode], *p->factors, mode, ai, c, ntc::RngStream(rng_state), &st);
    } else {
      ntc::s_nmc(p->views[mode], *p->factors, mode, p->factors->factors[mode], c,
                 ntc::RngStream(rng_state), &st);
    }
    if (accessed) *accessed += st.entries_accessed;
  });
}

int ref_objective(void* h, double lambda, double* out) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    if (!p->tensor || !p->factors) throw std::invalid_argument("ref_objective: no tensor");
    *out = ntc::objective(*p->tensor, *p->factors, lambda);
  });
}

int ref_relative_error(void* h, double* out) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    if (!p->tensor || !p->factors) throw std::invalid_argument("ref_relative_error: no tensor");
    *out = ntc::relative_error(*p->tensor, *p->factors);
  });
}

int ref_initial_factors(int order, const std::uint64_t* dims, std::uint64_t rank,
                        std::uint64_t seed, double* out) {
  return guarded([&] {
    std::vector<std::size_t> d(dims, dims + order);
    ntc::FactorSet f = ntc::initial_factors(d, rank, seed);
    std::size_t pos = 0;
    for (const auto& m : f.factors) {
      std::copy(m.data().begin(), m.data().end(), out + pos);
      pos += m.data().size();
    }
  });
}

// Runs the reference AO driver.  init/out are the N factors concatenated
// row-major; hist receives up to max_hist records of
// (epoch, objective, rel_error, wall_seconds, entries_accessed).
int ref_ao_ntc(void* h, const ref_ao_cfg* cfg, const double* init, double* out,
               double* hist, int max_hist, int* n_hist) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    if (!p->tensor) throw std::invalid_argument("ref_ao_ntc: no tensor");
    ntc::AoConfig c;
    c.rank = cfg->rank;
    c.lambda = cfg->lambda;
    c.c = cfg->c;
    c.max_inner = cfg->max_inner;
    c.max_epochs = cfg->max_epochs;
    c.term_tol = cfg->term_tol;
    c.seed = cfg->seed;
    c.threads = cfg->threads;
    c.chunk = cfg->chunk;
    c.power_iters = cfg->power_iters;
    c.power_tol = cfg->power_tol;
    c.eval_metrics = cfg->eval_metrics != 0;
    c.metrics_every = cfg->metrics_every;
    const std::size_t rank = cfg->rank ? cfg->rank : 1;
    ntc::FactorSet f = ntc::FactorSet::zeros(p->dims, rank);
    std::size_t pos = 0;
    for (std::size_t m = 0; m < p->dims.size(); ++m) {
      f.factors[m] = to_matrix(init + pos, p->dims[m], rank);
      f.momentum[m] = f.factors[m];
      pos += p->dims[m] * rank;
    }
    f.rank = cfg->rank;
    ntc::AoResult r = ntc::ao_ntc(*p->tensor, std::move(f), c);
    pos = 0;
    for (const auto& m : r.factors.factors) {
      std::copy(m.data().begin(), m.data().end(), out + pos);
      pos += m.data().size();
    }
    const int n = static_cast<int>(r.history.size());
    *n_hist = n;
    for (int i = 0; i < n && i < max_hist; ++i) {
      const auto& rec = r.history[i];
      hist[5 * i + 0] = rec.epoch;
      hist[5 * i + 1] = rec.objective;
      hist[5 * i + 2] = rec.rel_error;
      hist[5 * i + 3] = rec.wall_seconds;
      hist[5 * i + 4] = static_cast<double>(rec.entries_accessed);
    }
  });
}

// read_tns (tns_io.cpp:41-125): a problem handle, or NULL with the error text.
void* ref_read_tns(const char* path) {
  Problem* out = nullptr;
  int rc = guarded([&] {
    auto p = std::make_unique<Problem>();
    p->tensor.emplace(ntc::read_tns(path));
    p->dims = p->tensor->dims();
    p->views = ntc::build_mode_views(*p->tensor);
    out = p.release();
  });
  return rc == 0 ? out : nullptr;
}
int ref_order(void* h) { return static_cast<int>(static_cast<Problem*>(h)->dims.size()); }
void ref_dims(void* h, std::uint64_t* d) {
  auto* p = static_cast<Problem*>(h);
  for (std::size_t m = 0; m < p->dims.size(); ++m) d[m] = p->dims[m];
}
int ref_write_tns(void* h, const char* path) {
  return guarded([&] { ntc::write_tns(*static_cast<Problem*>(h)->tensor, path); });
}

// ---- per-row operators ----------------------------------------------------
// render_model (image.cpp:161-183) on a FactorSet built from host factors.
int ref_render_model(int order, const std::uint64_t* dims, std::uint64_t rank, const double* const* fac,
                     std::uint8_t* pixels) {
  return guarded([&] {
    std::vector<std::size_t> d(dims, dims + order);
    ntc::FactorSet f = ntc::FactorSet::zeros(d, rank);
    for (int m = 0; m < order; ++m) f.factors[m] = to_matrix(fac[m], d[m], rank);
    const ntc::Image img = ntc::render_model(f);
    std::copy(img.pixels.begin(), img.pixels.end(), pixels);
  });
}

int ref_power_method(std::uint64_t n, const double* hm, int iters, double tol, double* out) {
  return guarded([&] { *out = ntc::power_method(to_matrix(hm, n, n), iters, tol); });
}

int ref_row_step(std::uint64_t rank, const double* y, const double* a_prev, const double* grad,
                 double lipschitz, double lambda, double* a_new, double* y_new, double* beta) {
  return guarded([&] {
    *beta = ntc::row_step({y, rank}, {a_prev, rank}, {grad, rank}, lipschitz, lambda,
                          {a_new, rank}, {y_new, rank});
  });
}

// Gradient (w, z, grad) and Hessian of one row for an explicit pick list.
int ref_row_terms(void* h, int mode, std::uint64_t row, const std::uint32_t* picks,
                  std::uint64_t npicks, const double* y, double lambda, double* w, double* z,
                  double* grad, double* hess) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    if (!p->factors) throw std::invalid_argument("ref_row_terms: no factors");
    ntc::SampledRow s;
    s.row = row;
    s.picks.assign(picks, picks + npicks);
    const std::size_t rank = p->factors->rank;
    ntc::RowWorkspace ws;
    ws.resize(rank);
    ntc::row_gradient(p->views.at(mode), s, *p->factors, mode, {y, rank}, lambda, ws);
    std::copy(ws.w.begin(), ws.w.end(), w);
    std::copy(ws.z.begin(), ws.z.end(), z);
    std::copy(ws.grad.begin(), ws.grad.end(), grad);
    ntc::Matrix hm;
    ntc::row_hessian(p->views.at(mode), s, *p->factors, mode, lambda, hm);
    std::copy(hm.data().begin(), hm.data().end(), hess);
  });
}

}  // extern "C"
