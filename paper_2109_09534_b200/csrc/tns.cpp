// Parallel .tns reader / writer: the FROSTT-style text
// format of the reference's read_tns / write_tns (tns_io.cpp:41-142), same
// syntax, same diagnostics (path:line: message), same entry order, parsed by
// all host threads instead of one istringstream loop.
//
// Format (tns_io.hpp:9-16): one entry per line, N 1-based indices then the
// value; '#' starts a comment (a token beginning with '#' ends the line); an
// optional "# dims: I1 .. IN" header declares the dimensions (otherwise the
// componentwise maxima), and indices after a header are checked against it.
//
// Parallel scheme: the file is read once into memory and split at newlines
// into one chunk per thread.  Pass 1 (parallel) finds each chunk's line count,
// its header lines and its first entry line; a short sequential step turns
// these into global line numbers, the order N and the header in force at the
// start of every chunk; pass 2 (parallel) parses the entries.  Every chunk
// records its first error; the error with the smallest line number wins,
// which is the error the sequential reference reports.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "ntc_b200.h"

namespace {

thread_local std::string g_tns_err;

struct Header {
  uint64_t line;              // global line number
  std::vector<uint64_t> dims; // empty: not a dims header
  std::string error;          // parse error of the header itself
};

struct ChunkScan {
  uint64_t lines = 0;
  std::vector<std::pair<uint64_t, std::string>> headers;  // (local line, text after '#')
  uint64_t first_entry_line = 0;                          // local line, 0 = none
  size_t first_entry_fields = 0;
};

struct ChunkParse {
  std::vector<uint32_t> idx;
  std::vector<double> val;
  std::vector<uint64_t> maxima;
  uint64_t err_line = UINT64_MAX;
  std::string err;
};

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

// whitespace tokens of [b, e), stopping at a token that starts with '#'
inline void tokenize(const char* b, const char* e, std::vector<std::pair<const char*, const char*>>& out) {
  out.clear();
  const char* p = b;
  while (p < e) {
    while (p < e && is_ws(*p)) ++p;
    if (p >= e) break;
    if (*p == '#') break;
    const char* q = p;
    while (q < e && !is_ws(*q)) ++q;
    out.emplace_back(p, q);
    p = q;
  }
}

// the reference's header parse (tns_io.cpp:62-79) of the text after '#'
Header parse_header(uint64_t line, const std::string& text) {
  Header h;
  h.line = line;
  std::istringstream hs(text);
  std::string word;
  if (!(hs >> word && word == "dims:")) return h;  // an ordinary comment
  long long d = 0;
  std::vector<uint64_t> dims;
  while (hs >> d) {
    if (d <= 0) {
      h.error = "non-positive dimension in dims header";
      return h;
    }
    dims.push_back(static_cast<uint64_t>(d));
  }
  if (hs.fail() && !hs.eof()) {
    h.error = "bad dims header";
    return h;
  }
  if (dims.size() < 2) {
    h.error = "dims header needs at least 2 dimensions";
    return h;
  }
  h.dims = std::move(dims);
  return h;
}

}  // namespace

extern "C" {

const char* ntcb_tns_last_error(void) { return g_tns_err.c_str(); }

void ntcb_free(void* p) { std::free(p); }

int ntcb_tns_parse(const char* path_c, int* order_out, uint64_t* dims_out, uint64_t* nnz_out,
                   uint32_t** indices_out, double** values_out) {
  const std::string path(path_c ? path_c : "");
  try {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("read_tns: cannot open " + path);
    std::string buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    const char* data = buf.data();
    const size_t size = buf.size();
    unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    if (size < (1u << 20)) nt = 1;
    // chunk boundaries at line starts
    std::vector<size_t> cut(nt + 1, size);
    cut[0] = 0;
    for (unsigned t = 1; t < nt; ++t) {
      size_t p = size * t / nt;
      if (p < cut[t - 1]) p = cut[t - 1];
      while (p < size && data[p - 1] != '\n') ++p;
      cut[t] = p;
    }
    auto for_lines = [&](unsigned t, auto&& fn) {
      size_t p = cut[t];
      const size_t end = cut[t + 1];
      uint64_t ln = 0;
      while (p < end) {
        size_t q = p;
        while (q < end && data[q] != '\n') ++q;
        ++ln;
        if (!fn(ln, data + p, data + q)) return;
        p = q + 1;
      }
    };
    // ---- pass 1 ----
    std::vector<ChunkScan> scan(nt);
    {
      std::vector<std::thread> th;
      for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
          ChunkScan& cs = scan[t];
          std::vector<std::pair<const char*, const char*>> toks;
          for_lines(t, [&](uint64_t ln, const char* b, const char* e) {
            cs.lines = ln;
            const char* f = b;
            while (f < e && (*f == ' ' || *f == '\t' || *f == '\r')) ++f;
            if (f == e) return true;
            if (*f == '#') {
              cs.headers.emplace_back(ln, std::string(f + 1, e));
              return true;
            }
            if (cs.first_entry_line == 0) {
              tokenize(b, e, toks);
              if (!toks.empty()) {
                cs.first_entry_line = ln;
                cs.first_entry_fields = toks.size();
              }
            }
            return true;
          });
        });
      for (auto& x : th) x.join();
    }
    // ---- sequential: global line numbers, headers, order ----
    std::vector<uint64_t> base(nt + 1, 0);
    for (unsigned t = 0; t < nt; ++t) base[t + 1] = base[t] + scan[t].lines;
    std::vector<Header> headers;
    for (unsigned t = 0; t < nt; ++t)
      for (auto& hl : scan[t].headers) {
        Header h = parse_header(base[t] + hl.first, hl.second);
        if (!h.error.empty() || !h.dims.empty()) headers.push_back(std::move(h));
      }
    // order: from the first header or first entry line in file order
    uint64_t first_entry = UINT64_MAX;
    size_t first_fields = 0;
    for (unsigned t = 0; t < nt; ++t)
      if (scan[t].first_entry_line) {
        first_entry = base[t] + scan[t].first_entry_line;
        first_fields = scan[t].first_entry_fields;
        break;
      }
    uint64_t err_line = UINT64_MAX;
    std::string err;
    auto note = [&](uint64_t line, const std::string& m) {
      if (line < err_line) {
        err_line = line;
        err = m;
      }
    };
    size_t order = 0;
    {
      // replay the header/first-entry interplay of tns_io.cpp:62-95 in line order
      size_t hi = 0;
      bool entry_seen = false;
      while (hi < headers.size() || !entry_seen) {
        const uint64_t hl = hi < headers.size() ? headers[hi].line : UINT64_MAX;
        if (!entry_seen && first_entry < hl) {
          entry_seen = true;
          if (order == 0) {
            if (first_fields < 3) {
              note(first_entry, "expected at least 2 indices and a value");
              break;
            }
            order = first_fields - 1;
          }
          continue;
        }
        if (hl == UINT64_MAX) break;
        const Header& h = headers[hi++];
        if (!h.error.empty()) {
          note(h.line, h.error);
          break;
        }
        if (order != 0 && order != h.dims.size()) {
          note(h.line, "dims header order disagrees with entries");
          break;
        }
        order = h.dims.size();
      }
    }
    // ---- pass 2 ----
    std::vector<ChunkParse> parse(nt);
    if (order > 0) {
      std::vector<std::thread> th;
      for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
          ChunkParse& cp = parse[t];
          cp.maxima.assign(order, 0);
          // header in force at the chunk start, advanced as header lines pass
          size_t hi = 0;
          const std::vector<uint64_t>* decl = nullptr;
          while (hi < headers.size() && headers[hi].line <= base[t]) {
            if (headers[hi].error.empty()) decl = &headers[hi].dims;
            ++hi;
          }
          std::vector<std::pair<const char*, const char*>> toks;
          for_lines(t, [&](uint64_t ln, const char* b, const char* e) {
            const uint64_t g = base[t] + ln;
            while (hi < headers.size() && headers[hi].line <= g) {
              if (headers[hi].error.empty()) decl = &headers[hi].dims;
              ++hi;
            }
            const char* f = b;
            while (f < e && (*f == ' ' || *f == '\t' || *f == '\r')) ++f;
            if (f == e || *f == '#') return true;
            tokenize(b, e, toks);
            if (toks.empty()) return true;
            auto bad = [&](const std::string& m) {
              cp.err_line = g;
              cp.err = m;
              return false;
            };
            if (toks.size() != order + 1)
              return bad("expected " + std::to_string(order + 1) + " fields, got " +
                         std::to_string(toks.size()));
            for (size_t m = 0; m < order; ++m) {
              const std::string tok(toks[m].first, toks[m].second);
              long long v = 0;
              const auto [p, ec] = std::from_chars(toks[m].first, toks[m].second, v);
              if (ec != std::errc{} || p != toks[m].second) return bad("bad index '" + tok + "'");
              if (v < 1) return bad("indices are 1-based; got " + tok);
              if (static_cast<unsigned long long>(v) > std::numeric_limits<uint32_t>::max())
                return bad("index too large: " + tok);
              if (decl && static_cast<uint64_t>(v) > (*decl)[m])
                return bad("index " + tok + " exceeds declared dimension " + std::to_string((*decl)[m]));
              cp.idx.push_back(static_cast<uint32_t>(v - 1));
              cp.maxima[m] = std::max<uint64_t>(cp.maxima[m], static_cast<uint64_t>(v));
            }
            double val = 0.0;
            const std::string vt(toks[order].first, toks[order].second);
            const auto [p, ec] = std::from_chars(toks[order].first, toks[order].second, val);
            if (ec != std::errc{} || p != toks[order].second) return bad("bad value '" + vt + "'");
            if (!std::isfinite(val)) return bad("non-finite value");
            if (val < 0.0) return bad("negative value");
            cp.val.push_back(val);
            return true;
          });
        });
      for (auto& x : th) x.join();
      for (auto& cp : parse)
        if (cp.err_line != UINT64_MAX) note(cp.err_line, cp.err);
    }
    if (err_line != UINT64_MAX) throw std::runtime_error(path + ":" + std::to_string(err_line) + ": " + err);
    uint64_t nnz = 0;
    for (auto& cp : parse) nnz += cp.val.size();
    bool have_dims = false;
    std::vector<uint64_t> dims;
    for (auto& h : headers)
      if (h.error.empty()) {
        dims = h.dims;
        have_dims = true;
      }
    if (!have_dims && nnz == 0)
      throw std::runtime_error("read_tns: " + path + " has no entries and no dims header");
    if (!have_dims) {
      dims.assign(order, 0);
      for (auto& cp : parse)
        for (size_t m = 0; m < order; ++m) dims[m] = std::max(dims[m], cp.maxima[m]);
    }
    if (dims.size() > NTCB_MAX_ORDER) throw std::invalid_argument("read_tns: order exceeds 8");
    uint32_t* idx = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * std::max<uint64_t>(nnz * dims.size(), 1)));
    double* val = static_cast<double*>(std::malloc(sizeof(double) * std::max<uint64_t>(nnz, 1)));
    uint64_t pos = 0;
    for (auto& cp : parse) {
      std::memcpy(idx + pos * dims.size(), cp.idx.data(), sizeof(uint32_t) * cp.idx.size());
      std::memcpy(val + pos, cp.val.data(), sizeof(double) * cp.val.size());
      pos += cp.val.size();
    }
    *order_out = static_cast<int>(dims.size());
    for (size_t m = 0; m < dims.size(); ++m) dims_out[m] = dims[m];
    *nnz_out = nnz;
    *indices_out = idx;
    *values_out = val;
    return NTCB_OK;
  } catch (const std::invalid_argument& e) {
    g_tns_err = e.what();
    return NTCB_EINVAL;
  } catch (const std::exception& e) {
    g_tns_err = e.what();
    return NTCB_ERUNTIME;
  }
}

// write_tns (tns_io.cpp:127-142): "# dims:" header, 1-based indices, %.17g.
int ntcb_tns_write(const char* path_c, int order, const uint64_t* dims, uint64_t nnz,
                   const uint32_t* indices, const double* values) {
  const std::string path(path_c ? path_c : "");
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) {
    g_tns_err = "write_tns: cannot open " + path;
    return NTCB_ERUNTIME;
  }
  std::string out = "# dims:";
  for (int m = 0; m < order; ++m) out += " " + std::to_string(dims[m]);
  out += "\n";
  char buf[64];
  for (uint64_t e = 0; e < nnz; ++e) {
    for (int m = 0; m < order; ++m) {
      out += std::to_string(static_cast<uint64_t>(indices[e * order + m]) + 1);
      out += ' ';
    }
    std::snprintf(buf, sizeof buf, "%.17g", values[e]);
    out += buf;
    out += '\n';
    if (out.size() > (1u << 24)) {
      std::fwrite(out.data(), 1, out.size(), f);
      out.clear();
    }
  }
  const bool ok = std::fwrite(out.data(), 1, out.size(), f) == out.size();
  if (std::fclose(f) != 0 || !ok) {
    g_tns_err = "write_tns: write failed for " + path;
    return NTCB_ERUNTIME;
  }
  return NTCB_OK;
}

}  // extern "C"
