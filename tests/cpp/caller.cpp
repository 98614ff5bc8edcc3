// A reference-side C++ caller of the B200 library through the wrappers in
// include/gridhop_b200.hpp (the reference's estimator signatures and
// exception types). Reads a scene from stdin, prints one JSON object per
// check; tests/test_cpp_caller.py compares them with the fp64 oracle.
#include <cmath>
#include <cstdio>
#include <iostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "gridhop_b200.hpp"

namespace gb = gridhop::b200;

template <class E, class F>
std::string expect_throw(F&& f) {
  try {
    f();
  } catch (const E& e) {
    return e.what();
  } catch (const std::exception& e) {
    return std::string("WRONG TYPE: ") + e.what();
  }
  return "NO THROW";
}

std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char ch : s) o += (ch == '"' || ch == '\\') ? std::string("\\") + ch : std::string(1, ch);
  return o + "\"";
}

template <class T>
void print_list(const char* key, const std::vector<T>& v) {
  std::cout << "{\"" << key << "\": [";
  for (size_t i = 0; i < v.size(); ++i) std::cout << (i ? ", " : "") << v[i];
  std::cout << "]}\n";
}

int main() {
  gb::Scene s;
  int P = 0, T = 0;
  uint64_t seed = 0;
  double snr = 0.0;
  std::cin >> s.n_samples >> s.os_range >> s.bandwidth >> P;
  s.tx.resize(3 * P);
  s.rx.resize(3 * P);
  for (auto& v : s.tx) std::cin >> v;
  for (auto& v : s.rx) std::cin >> v;
  for (int d = 0; d < 3; ++d) std::cin >> s.grid.origin[d];
  for (int d = 0; d < 3; ++d) std::cin >> s.grid.spacing[d];
  for (int d = 0; d < 3; ++d) std::cin >> s.grid.n[d];
  gb::SceneModel model{};
  std::cin >> seed >> snr >> T;
  model.seed = seed;
  model.n_targets = 1;
  model.dims = 2;
  for (int d = 0; d < 3; ++d) std::cin >> model.area_lo[d];
  for (int d = 0; d < 3; ++d) std::cin >> model.area_hi[d];
  model.amp_mode = 1;
  model.snr_mode = 0;
  model.snr_db = snr;
  if (!std::cin) {
    std::cerr << "bad input\n";
    return 2;
  }

  gb::Context ctx(0);
  // synthesize_frame + add_noise on the device; hop and direct estimates
  auto [frames, truth] = gb::synthesize_frame(ctx, s, model, 0, T, /*wrap=*/true);
  gb::HopTable table = gb::precompute_hop_table(ctx, s, gb::InterpScheme::poly3, /*wrap=*/true);
  const gb::Estimates hop = gb::hop_estimate(ctx, table, frames, T);
  const gb::Estimates dir = gb::direct_estimate(ctx, s, frames, T);
  print_list("hop", hop.bin);
  print_list("direct", dir.bin);
  const std::vector<double> map = gb::hop_decision_map(ctx, table, frames, T);
  const double one = gb::hop_location_decision(ctx, table,
                                               std::vector<gb::cplx>(frames.begin(),
                                                                     frames.begin() + P * s.n_samples),
                                               static_cast<int>(hop.bin[0]));
  std::printf("{\"map_peak_t0\": %.9g, \"single_bin_t0\": %.9g}\n", map[size_t(hop.bin[0])], one);
  const auto spec = gb::fast_time_spectra(ctx, frames, T, P, s.n_samples, s.os_range);
  std::printf("{\"spectrum_t0_p0_b0\": [%.9g, %.9g]}\n", spec[0].real(), spec[0].imag());
  // noise on noiseless frames equals the synthesis' own noise draws
  gb::SceneModel quiet = model;
  quiet.snr_mode = 2;
  auto [clean, truth2] = gb::synthesize_frame(ctx, s, quiet, 0, T, true);
  gb::add_noise(ctx, clean, T, P, s.n_samples, snr, seed, 0);
  double dmax = 0.0;
  for (size_t i = 0; i < clean.size(); ++i) dmax = std::max(dmax, std::abs(clean[i] - frames[i]));
  std::printf("{\"add_noise_max_diff\": %.3g}\n", dmax);
  // fit_atom known answers (test_interp.cpp:76-103)
  const gb::AtomFit nf = gb::fit_atom(ctx, 16, 2, 3.30, gb::InterpScheme::nearest);
  const gb::AtomFit lf = gb::fit_atom(ctx, 16, 2, 3.30, gb::InterpScheme::linear);
  std::printf("{\"fit_nearest\": [%u, %.12g], \"fit_linear\": [%u, %u, %.12g, %.12g]}\n", nf.idx[0],
              nf.coef[0].real(), lf.idx[0], lf.idx[1], lf.coef[0].real(), lf.coef[1].real());
  // the reference's exception types and messages
  std::vector<gb::cplx> short_frames(frames.begin(), frames.end() - 1);
  std::cout << "{\"shape\": "
            << json_str(expect_throw<std::invalid_argument>(
                   [&] { gb::hop_estimate(ctx, table, short_frames, T); }))
            << "}\n";
  gb::Scene far = s;
  for (int d = 0; d < 2; ++d) far.grid.origin[d] = -1000.0;
  std::cout << "{\"window\": "
            << json_str(expect_throw<std::runtime_error>(
                   [&] { gb::precompute_hop_table(ctx, far, gb::InterpScheme::nearest, false); }))
            << "}\n";
  gb::SceneModel on_station = model;
  for (int d = 0; d < 3; ++d) on_station.area_lo[d] = on_station.area_hi[d] = s.rx[d];
  on_station.dims = 2;
  std::cout << "{\"degenerate\": "
            << json_str(expect_throw<std::domain_error>(
                   [&] { gb::synthesize_frame(ctx, s, on_station, 0, 2, true); }))
            << "}\n";
  std::cout << "{\"bad_range\": "
            << json_str(expect_throw<std::invalid_argument>(
                   [&] { gb::fit_atom(ctx, 16, 2, NAN, gb::InterpScheme::nearest); }))
            << "}\n";
  // run_monte_carlo with a TableSource supplying the table built above
  gb::Scenario sc;
  sc.scene = s;
  sc.model = model;
  sc.scheme = gb::InterpScheme::poly3;
  sc.wrap = true;
  sc.algorithms = {gb::Algorithm::direct, gb::Algorithm::hop};
  sc.trials = T;
  int source_calls = 0;
  gb::TableSource src = [&](double density, const gh_grid&) {
    ++source_calls;
    (void)density;
    return std::make_pair(gb::precompute_hop_table(ctx, s, gb::InterpScheme::poly3, true),
                          int64_t(12345));
  };
  const auto cells = gb::run_monte_carlo(ctx, sc, nullptr, src);
  std::printf("{\"mc_cells\": %zu, \"source_calls\": %d, \"hop_offline_ns\": %.0f, "
              "\"direct_hits_1m\": %.0f, \"hop_hits_1m\": %.0f, \"hop_rmse\": %.9g}\n",
              cells.size(), source_calls, cells[1].offline_ms * 1e6, cells[0].hits[4],
              cells[1].hits[4], cells[1].rmse_m);
  return 0;
}
