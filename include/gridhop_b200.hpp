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

#include <complex>
#include <cstdint>
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

// hop_estimate location stage (hopping.hpp:35-38) for a batch of trials:
// frames = T FrameSets of P receivers x N complex samples (Mc = 1),
// trial-major [T][P][N] — the reference's FrameSet element type.
inline Estimates hop_estimate(Context& ctx, const HopTable& table, const std::vector<cplx>& frames,
                              int n_trials, Combine combine = Combine::power) {
  if (n_trials < 0 || frames.size() % (n_trials ? size_t(n_trials) : 1) != 0)
    throw std::invalid_argument("hop: frame shape mismatch");
  Estimates e;
  e.bin.resize(n_trials);
  e.value.resize(n_trials);
  check(gh_hop_estimate(ctx.get(), table.get(), reinterpret_cast<const double*>(frames.data()),
                        n_trials, static_cast<int32_t>(combine), e.bin.data(), e.value.data()));
  return e;
}

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
