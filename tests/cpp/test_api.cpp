// C++ host API smoke test (include/ntcb.hpp over libntcb.so): the reference's
// call pattern of test_ao.cpp:151-183 (an AO sweep equals the mode-by-mode
// replay through s_nmc with sweep_stream) and its exception types.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "ntcb.hpp"

static int fails = 0;
#define EXPECT(cond)                                         \
  do {                                                       \
    if (!(cond)) {                                           \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); \
      ++fails;                                               \
    }                                                        \
  } while (0)

int main() {
  const std::vector<std::size_t> dims{6, 5, 4};
  std::vector<std::uint32_t> idx;
  std::vector<double> vals;
  std::uint64_t s = 12345;
  for (std::uint32_t i = 0; i < 6; ++i)
    for (std::uint32_t j = 0; j < 5; ++j)
      for (std::uint32_t k = 0; k < 4; ++k) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        if ((s >> 60) < 10) {  // ~60% density
          idx.insert(idx.end(), {i, j, k});
          vals.push_back(static_cast<float>(((s >> 20) & 0xffff) / 65536.0 * 2.0));
        }
      }
  ntcb::AoConfig cfg;
  cfg.rank = 3;
  cfg.c = 0.5;
  cfg.seed = 11;
  cfg.max_epochs = 1e-9;  // stop right after the first sweep

  ntcb::Solver ao;
  ao.load(dims, idx, vals);
  ao.initial_factors(3, cfg.seed);
  const auto hist = ao.ao_ntc(cfg);
  EXPECT(hist.size() == 2);

  ntcb::Solver replay;
  replay.load(dims, idx, vals);
  replay.initial_factors(3, cfg.seed);
  for (int i = 0; i < 3; ++i) replay.s_nmc(i, nullptr, cfg.nmc(), ntcb::sweep_stream(cfg.seed, 0, i));
  for (int i = 0; i < 3; ++i) EXPECT(replay.factor(i) == ao.factor(i));

  bool threw = false;
  try {
    ntcb::NmcConfig bad;
    bad.lambda = 0.0;
    replay.s_nmc(0, nullptr, bad, ntcb::RngStream(1));
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()) == "NmcConfig: lambda must be > 0";
  }
  EXPECT(threw);
  threw = false;
  try {
    ntcb::Solver t;
    t.load({2, 2}, {0, 1, 0, 1}, {1.0, 2.0});
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()) == "SparseTensor: duplicate index (1,2)";
  }
  EXPECT(threw);
  const double rel = ao.relative_error();
  EXPECT(std::isfinite(rel) && rel > 0.0);
  threw = false;
  try {
    (void)ao.render_model();  // 6 x 5 x 4 tensor: not an H x W x 3 factorization
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()) == "render_model: expects an H x W x 3 factorization";
  }
  EXPECT(threw);
  ntcb_tuning tn = ao.tuning();
  EXPECT(tn.update_wpc == 4 && tn.nat_pad == -1);
  tn.update_wpc = 2;
  ao.set_tuning(tn);
  EXPECT(ao.tuning().update_wpc == 2);
  std::printf("%s (%d failures)\n", fails ? "FAILED" : "ok", fails);
  return fails ? 1 : 0;
}
