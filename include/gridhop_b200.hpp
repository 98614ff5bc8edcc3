// gridhop_b200.hpp — C++ wrappers over the C ABI, keeping the reference
// library's estimator interfaces and exception behaviour
// (/root/reference/proj/core/include/gridhop/{interp,hopping,direct,synth}.hpp).
//
// Header-only; link against libgridhop_b200.so. Status codes are rethrown as
// the exception types the reference throws (std::invalid_argument,
// std::runtime_error, std::domain_error) with the library's message, e.g.
// "hop table: sensed range outside [0, n_samples) at ..." (interp.cpp:198),
// "scene outside unambiguous window" (synth.cpp:29),
// "degenerate geometry: target coincides with a station" (model.cpp:50).
#pragma once

#include <algorithm>
#include <complex>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gridhop_b200.h"

namespace gridhop {
namespace b200 {

using cplx = std::complex<double>;

enum class InterpScheme { nearest = GH_NEAREST, linear = GH_LINEAR, poly3 = GH_POLY3, polar = GH_POLAR };
enum class Combine { power = GH_POWER, magnitude = GH_MAGNITUDE };

inline void check(int status) {
  if (status == GH_OK) return;
  const std::string msg = gh_last_error();
  switch (status) {
    case GH_EINVAL: throw std::invalid_argument(msg);
    case GH_EDOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// WaveformConfig + SceneGeometry (model.hpp:21-50), generalised to TX-RX pairs
struct Scene {
  int n_samples = 128;
  int os_range = 4;
  double bandwidth = 250.0e6;
  double c = 299792458.0;
  std::vector<double> tx;  // [P][3]
  std::vector<double> rx;  // [P][3]
  gh_grid grid{};          // LocationGrid (model.hpp:77-92), x fastest

  int n_pairs() const { return static_cast<int>(tx.size() / 3); }
  int64_t n_bins() const { return int64_t(grid.n[0]) * grid.n[1] * grid.n[2]; }
  double range_scale() const { return bandwidth / c; }  // model.hpp:36
  gh_wave wave() const {
    return gh_wave{n_samples, os_range, range_scale(), n_pairs(), tx.data(), rx.data()};
  }
};

class Context {
 public:
  explicit Context(int device = 0) { check(gh_ctx_create(device, &h_)); }
  ~Context() { if (h_) gh_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  gh_ctx* get() const { return h_; }
  void synchronize() const { check(gh_ctx_synchronize(h_)); }

 private:
  gh_ctx* h_ = nullptr;
};

// HopTable (interp.hpp:44-60), resident on the device
class HopTable {
 public:
  HopTable(gh_table* h) : h_(h) {
    check(gh_table_info(h_, &n_bins, &n_rx, &k, &n_fft, &max_residual));
  }
  ~HopTable() { if (h_) gh_table_destroy(h_); }
  HopTable(HopTable&& o) noexcept { *this = std::move(o); }
  HopTable& operator=(HopTable&& o) noexcept {
    std::swap(h_, o.h_);
    n_bins = o.n_bins; n_rx = o.n_rx; k = o.k; n_fft = o.n_fft; max_residual = o.max_residual;
    return *this;
  }
  HopTable(const HopTable&) = delete;
  gh_table* get() const { return h_; }

  // the operator in the reference layout [bin][receiver][K] (entry_offset)
  std::pair<std::vector<uint32_t>, std::vector<cplx>> download() const {
    std::vector<uint32_t> idx(size_t(n_bins) * n_rx * k);
    std::vector<cplx> coef(idx.size());
    check(gh_table_download(h_, idx.data(), reinterpret_cast<double*>(coef.data())));
    return {std::move(idx), std::move(coef)};
  }

  int64_t n_bins = 0;
  int32_t n_rx = 0, k = 0, n_fft = 0;
  double max_residual = 0.0;

 private:
  gh_table* h_ = nullptr;
};

// precompute_hop_table (interp.hpp:65-67), built on the device in fp64;
// wrap = true accepts aliasing scenes (the atoms are periodic, interp.cpp:39-44)
inline HopTable precompute_hop_table(Context& ctx, const Scene& s, InterpScheme scheme,
                                     bool wrap = false) {
  const gh_wave w = s.wave();
  gh_table* t = nullptr;
  check(gh_table_build(ctx.get(), &w, &s.grid, static_cast<int32_t>(scheme), wrap ? 1 : 0, &t));
  return HopTable(t);
}

// load_hop_table analogue: a host operator in the reference layout
inline HopTable upload_hop_table(Context& ctx, const Scene& s, InterpScheme scheme,
                                 const std::vector<uint32_t>& idx, const std::vector<cplx>& coef) {
  const gh_wave w = s.wave();
  gh_table* t = nullptr;
  check(gh_table_upload(ctx.get(), &w, &s.grid, static_cast<int32_t>(scheme), idx.data(),
                        coef.empty() ? nullptr : reinterpret_cast<const double*>(coef.data()), &t));
  return HopTable(t);
}

// scene_hash (model.hpp / model.cpp:135-166) of a single-TX 2-D scene: the
// key GHT1 files are bound to. rx_xy = {x0, y0, x1, y1, ...}.
inline uint64_t scene_hash(int n_chirps, int n_samples, double f0, double bandwidth,
                           double chirp_duration, const double tx_xy[2],
                           const std::vector<double>& rx_xy) {
  return gh_scene_hash(static_cast<int32_t>(rx_xy.size() / 2), n_chirps, n_samples, f0, bandwidth,
                       chirp_duration, tx_xy, rx_xy.data());
}

// save_hop_table (interp.hpp:72): the device operator as a GHT1 file
inline void save_hop_table(const std::string& path, const HopTable& table, uint64_t scene_hash) {
  check(gh_table_save(table.get(), path.c_str(), scene_hash));
}

// load_hop_table (interp.hpp:76-77): refuses files built for another scene
// or grid ("stale hop table"), then uploads
inline HopTable load_hop_table(Context& ctx, const std::string& path, const Scene& s,
                               uint64_t scene_hash) {
  const gh_wave w = s.wave();
  gh_table* t = nullptr;
  check(gh_table_load(ctx.get(), path.c_str(), &w, &s.grid, scene_hash, &t));
  return HopTable(t);
}

// Capture (frame_io.hpp:17-21) with frames flattened trial-major:
// frames[((t * n_rx + q) * n_chirps + m) * n_samples + s]
struct Capture {
  gh_mrf1_header header{};
  std::vector<double> rx;     // {x0, y0, x1, y1, ...}
  std::vector<cplx> frames;
};

// read_frames (frame_io.hpp:27): validates like the reference, throws its
// exception types and texts
inline Capture read_frames(const std::string& path) {
  Capture cap;
  check(gh_mrf1_read(path.c_str(), &cap.header, nullptr, 0, nullptr, 0));
  cap.rx.resize(2 * size_t(cap.header.n_rx));
  cap.frames.resize(size_t(cap.header.n_frames) * cap.header.n_rx * cap.header.n_chirps *
                    cap.header.n_samples);
  check(gh_mrf1_read(path.c_str(), &cap.header, cap.rx.data(), cap.header.n_rx,
                     reinterpret_cast<double*>(cap.frames.data()),
                     static_cast<int64_t>(cap.frames.size())));
  return cap;
}

// write_frames (frame_io.hpp:23-25)
inline void write_frames(const std::string& path, const Capture& cap) {
  if (cap.rx.size() != 2 * size_t(cap.header.n_rx))
    throw std::invalid_argument(path + ": frame/receiver count mismatch");
  if (cap.frames.size() != size_t(cap.header.n_frames) * cap.header.n_rx *
                               cap.header.n_chirps * cap.header.n_samples)
    throw std::invalid_argument(path + ": frame shape mismatch");
  check(gh_mrf1_write(path.c_str(), &cap.header, cap.rx.data(),
                      reinterpret_cast<const double*>(cap.frames.data())));
}

struct Estimates {
  std::vector<int64_t> bin;  // per trial, argmax_index rule (direct.cpp:55-62)
  std::vector<double> value;
};

// the table's waveform: (n_samples, os_range)
inline std::pair<int, int> table_geometry(const HopTable& table) {
  int32_t n = 0, os = 0;
  check(gh_table_geometry(table.get(), &n, &os, nullptr));
  return {n, os};
}

// frames of T trials x P pairs x N samples, trial-major: the reference's
// FrameSet (synth.hpp:12) with Mc = 1, one FrameSet per trial
inline void check_frames(const std::vector<cplx>& frames, int n_trials, int n_pairs,
                         int n_samples) {
  if (n_trials < 0 || frames.size() != size_t(n_trials) * size_t(n_pairs) * size_t(n_samples))
    throw std::invalid_argument("hop: frame shape mismatch");  // hopping.cpp:251
}

// hop_estimate location stage (hopping.hpp:35-38) for a batch of trials:
// frames = T FrameSets of P receivers x N complex samples (Mc = 1),
// trial-major [T][P][N] — the reference's FrameSet element type.
inline Estimates hop_estimate(Context& ctx, const HopTable& table, const std::vector<cplx>& frames,
                              int n_trials, Combine combine = Combine::power) {
  check_frames(frames, n_trials, table.n_rx, table_geometry(table).first);
  Estimates e;
  e.bin.resize(n_trials);
  e.value.resize(n_trials);
  check(gh_hop_estimate(ctx.get(), table.get(), reinterpret_cast<const double*>(frames.data()),
                        n_trials, static_cast<int32_t>(combine), e.bin.data(), e.value.data()));
  return e;
}

// multi-target form (BASELINE c3): the k best local maxima per trial,
// [T][k] row-major, bin -1 when a trial has fewer maxima
inline Estimates hop_estimate_topk(Context& ctx, const HopTable& table,
                                   const std::vector<cplx>& frames, int n_trials, int k,
                                   Combine combine = Combine::power) {
  check_frames(frames, n_trials, table.n_rx, table_geometry(table).first);
  Estimates e;
  e.bin.resize(size_t(n_trials) * k);
  e.value.resize(size_t(n_trials) * k);
  check(gh_hop_estimate_topk(ctx.get(), table.get(), reinterpret_cast<const double*>(frames.data()),
                             n_trials, static_cast<int32_t>(combine), k, e.bin.data(),
                             e.value.data()));
  return e;
}

// fast_time_spectra (hopping.hpp:14): zero-padded forward FFT of every
// (trial, pair) row, [T][P][N] -> [T][P][os * N]
inline std::vector<cplx> fast_time_spectra(Context& ctx, const std::vector<cplx>& frames,
                                           int n_trials, int n_pairs, int n_samples,
                                           int os_range) {
  check_frames(frames, n_trials, n_pairs, n_samples);
  std::vector<cplx> out(size_t(n_trials) * n_pairs * n_samples * os_range);
  check(gh_spectra(ctx.get(), reinterpret_cast<const double*>(frames.data()), n_trials, n_pairs,
                   n_samples, os_range, reinterpret_cast<double*>(out.data())));
  return out;
}

// hop_decision_map (hopping.hpp:22): [T][G] decision values
inline std::vector<double> hop_decision_map(Context& ctx, const HopTable& table,
                                            const std::vector<cplx>& frames, int n_trials,
                                            Combine combine = Combine::power) {
  check_frames(frames, n_trials, table.n_rx, table_geometry(table).first);
  std::vector<double> map(size_t(n_trials) * size_t(table.n_bins));
  check(gh_hop_map(ctx.get(), table.get(), reinterpret_cast<const double*>(frames.data()), n_trials,
                   static_cast<int32_t>(combine), map.data()));
  return map;
}

// hop_location_decision (hopping.hpp:18): one bin of one trial's map
inline double hop_location_decision(Context& ctx, const HopTable& table,
                                    const std::vector<cplx>& frame, int bin,
                                    Combine combine = Combine::power) {
  if (bin < 0 || bin >= table.n_bins) throw std::invalid_argument("hop: bin out of range");
  return hop_decision_map(ctx, table, frame, 1, combine)[size_t(bin)];
}

// location_decision_map (direct.hpp:19-23): the direct method's [T][G] map
inline std::vector<double> location_decision_map(Context& ctx, const Scene& s,
                                                 const std::vector<cplx>& frames, int n_trials,
                                                 Combine combine = Combine::power) {
  check_frames(frames, n_trials, s.n_pairs(), s.n_samples);
  const gh_wave w = s.wave();
  std::vector<double> map(size_t(n_trials) * size_t(s.n_bins()));
  check(gh_direct_map(ctx.get(), &w, &s.grid, reinterpret_cast<const double*>(frames.data()),
                      n_trials, static_cast<int32_t>(combine), map.data()));
  return map;
}

// direct_estimate location stage (direct.hpp:37-39): per-trial argmax
inline Estimates direct_estimate(Context& ctx, const Scene& s, const std::vector<cplx>& frames,
                                 int n_trials, Combine combine = Combine::power) {
  check_frames(frames, n_trials, s.n_pairs(), s.n_samples);
  const gh_wave w = s.wave();
  Estimates e;
  e.bin.resize(n_trials);
  e.value.resize(n_trials);
  check(gh_direct_estimate(ctx.get(), &w, &s.grid, reinterpret_cast<const double*>(frames.data()),
                           n_trials, static_cast<int32_t>(combine), e.bin.data(), e.value.data()));
  return e;
}

// AtomFit (interp.hpp:32-37) and fit_atom (interp.hpp:41), fitted on the
// device with the table builder's fp64 code
struct AtomFit {
  std::vector<uint32_t> idx;
  std::vector<cplx> coef;
  double residual = 0.0;
};
inline AtomFit fit_atom(Context& ctx, int n_samples, int os, double r, InterpScheme scheme) {
  uint32_t idx[3];
  double coef[6], res = 0.0;
  check(gh_fit_atom(ctx.get(), n_samples, os, &r, 1, static_cast<int32_t>(scheme), idx, coef, &res));
  const int k = scheme == InterpScheme::nearest ? 1 : (scheme == InterpScheme::linear ? 2 : 3);
  AtomFit f;
  for (int j = 0; j < k; ++j) {
    f.idx.push_back(idx[j]);
    f.coef.emplace_back(coef[2 * j], coef[2 * j + 1]);
  }
  f.residual = res;
  return f;
}

// The Monte-Carlo scene model (sample_scene, montecarlo.cpp:48-66, with the
// BASELINE extensions): gh_campaign
using SceneModel = gh_campaign;

// synthesize_frame (synth.hpp:26-27) of trials [trial0, trial0 + T) of the
// scene model (noise per its SNR model, snr_mode 2 = noiseless): frames
// [T][P][N] and truths [T][K][3]
inline std::pair<std::vector<cplx>, std::vector<double>> synthesize_frame(
    Context& ctx, const Scene& s, const SceneModel& model, uint64_t trial0, int n_trials,
    bool wrap = false) {
  const gh_wave w = s.wave();
  std::vector<cplx> frames(size_t(n_trials) * s.n_pairs() * s.n_samples);
  std::vector<double> truth(size_t(n_trials) * model.n_targets * 3);
  check(gh_synth(ctx.get(), &w, &model, trial0, n_trials, wrap ? 1 : 0,
                 reinterpret_cast<double*>(frames.data()), truth.data()));
  return {std::move(frames), std::move(truth)};
}

// add_noise (synth.hpp:29-36): NoiseSpec{snr_db, alpha_ref = 1, seed},
// trials [trial0, trial0 + T) of frames [T][P][N]
inline void add_noise(Context& ctx, std::vector<cplx>& frames, int n_trials, int n_pairs,
                      int n_samples, double snr_db, uint64_t seed, uint64_t trial0) {
  check_frames(frames, n_trials, n_pairs, n_samples);
  check(gh_add_noise(ctx.get(), reinterpret_cast<double*>(frames.data()), n_trials, n_pairs,
                     n_samples, seed, trial0, snr_db));
}

// ---- Monte-Carlo campaign (montecarlo.hpp:43-77)

enum class Algorithm { indirect = GH_ALGO_INDIRECT, direct = GH_ALGO_DIRECT, hop = GH_ALGO_HOP };

// Scenario (scenario.hpp:22-52) restricted to what the device campaign reads
struct Scenario {
  Scene scene;
  SceneModel model{};
  InterpScheme scheme = InterpScheme::nearest;
  bool wrap = false;
  Combine combine = Combine::power;
  std::vector<Algorithm> algorithms = {Algorithm::indirect, Algorithm::direct, Algorithm::hop};
  std::vector<double> snr_db;      // empty: the model's SNR; NaN: noiseless
  std::vector<double> densities;   // empty: {1}
  std::vector<double> thresholds;  // empty: 0.2 .. 3.0 m
  int64_t trials = 1;
  int topk = 1;
  std::string trial_csv, summary_csv;
};

using CellStats = gh_cell_stats;

// TableSource (montecarlo.hpp:43-45): the hop table of a density cell plus
// the offline nanoseconds to report (e.g. load_hop_table of a cached file)
using TableSource = std::function<std::pair<HopTable, int64_t>(double density, const gh_grid& grid)>;

namespace detail {
struct SourceState {
  const TableSource* fn;
  std::vector<HopTable> keep;  // tables stay alive until the campaign returns
};
inline gh_table* table_source_trampoline(void* user, double density, const gh_grid* grid,
                                         int64_t* offline_ns) {
  auto* st = static_cast<SourceState*>(user);
  try {
    auto got = (*st->fn)(density, *grid);
    *offline_ns = got.second;
    st->keep.push_back(std::move(got.first));
    return st->keep.back().get();
  } catch (...) {
    return nullptr;
  }
}
}  // namespace detail

// run_monte_carlo (montecarlo.hpp:51-53): every (density, SNR, algorithm)
// cell on the device; with a communicator the trials are sharded over its
// ranks (one process per GPU) and the statistics all-reduced.
inline std::vector<CellStats> run_monte_carlo(Context& ctx, const Scenario& sc,
                                              gh_comm* comm = nullptr,
                                              const TableSource& tables = {}) {
  std::vector<int32_t> algos;
  for (Algorithm a : sc.algorithms) algos.push_back(static_cast<int32_t>(a));
  gh_campaign_desc d{};
  d.wave = sc.scene.wave();
  d.grid = sc.scene.grid;
  d.scene = sc.model;
  d.scheme = static_cast<int32_t>(sc.scheme);
  d.wrap = sc.wrap ? 1 : 0;
  d.combine = static_cast<int32_t>(sc.combine);
  d.n_algorithms = static_cast<int32_t>(algos.size());
  d.algorithms = algos.data();
  d.n_snr = static_cast<int32_t>(sc.snr_db.size());
  d.snr_db = sc.snr_db.data();
  d.n_density = static_cast<int32_t>(sc.densities.size());
  d.density = sc.densities.data();
  d.n_thresholds = static_cast<int32_t>(sc.thresholds.size());
  d.thresholds_m = sc.thresholds.data();
  d.n_trials = sc.trials;
  d.topk = sc.topk;
  d.trial_csv = sc.trial_csv.empty() ? nullptr : sc.trial_csv.c_str();
  d.summary_csv = sc.summary_csv.empty() ? nullptr : sc.summary_csv.c_str();
  detail::SourceState st{&tables, {}};
  st.keep.reserve(std::max<size_t>(1, sc.densities.size()));
  if (tables) {
    d.table_source = &detail::table_source_trampoline;
    d.table_source_user = &st;
  }
  const size_t cells = std::max<size_t>(1, sc.densities.size()) *
                       std::max<size_t>(1, sc.snr_db.size()) * algos.size();
  std::vector<CellStats> out(cells);
  int32_t n = 0;
  check(gh_campaign_run(ctx.get(), comm, &d, out.data(), static_cast<int32_t>(cells), &n));
  out.resize(size_t(n));
  return out;
}

// hit_ratio (montecarlo.hpp:57-59) of a cell at its j-th threshold
inline double hit_ratio(const CellStats& c, int j) { return c.hit_ratio[j]; }

// argmax_index (direct.hpp:43): first strict maximum
inline int argmax_index(const std::vector<double>& v) {
  if (v.empty()) throw std::invalid_argument("argmax of empty scan");
  int best = 0;
  for (int i = 1; i < static_cast<int>(v.size()); ++i)
    if (v[i] > v[best]) best = i;
  return best;
}

}  // namespace b200
}  // namespace gridhop
