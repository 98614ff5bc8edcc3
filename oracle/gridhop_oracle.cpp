// gridhop_oracle.cpp — CPU fp64 restatement of the reference hot path.
//
// TEST INFRASTRUCTURE ONLY (see gridhop_oracle.h). Compiled with
// -ffp-contract=off so every product below rounds exactly as written; the
// device table builder mirrors the same operation order with __dmul_rn /
// __dadd_rn so mapping indices come out bit-identical.
//
// Reference anchors (paths under /root/reference/proj/core):
//   rng        include/gridhop/rng.hpp:11-52
//   geometry   src/model.cpp:45-52 (sensed_range), 108-111 (grid point)
//   synth      src/synth.cpp:10-57, src/montecarlo.cpp:48-66 (scene draw)
//   fft        src/fft.cpp:132-146 / include/gridhop/fft.hpp:7-10
//   fit_atom   src/interp.cpp:21-154; table src/interp.cpp:156-223
//   hop scan   src/hopping.cpp:59-117
//   direct     src/direct.cpp:20-35 (conj_atom), 90-144 (decision map)
//   argmax     src/direct.cpp:55-62
//   campaign   src/montecarlo.cpp:99-179
#include "gridhop_oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using cplx = std::complex<double>;
constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr uint64_t kSceneTag = 0x53434E;  // montecarlo.cpp:22

thread_local std::string g_err;

struct domain_error_t : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const domain_error_t& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// parallel.hpp:15-46: shared counter, first exception rethrown.
template <class Fn>
void parallel_for(int64_t n, int n_threads, Fn&& fn) {
  if (n <= 0) return;
  if (n_threads < 1) n_threads = 1;
  const int workers = static_cast<int>(std::min<int64_t>(n_threads, n));
  if (workers == 1) {
    for (int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int64_t> next{0};
  std::mutex mu;
  std::exception_ptr first;
  auto body = [&] {
    for (;;) {
      const int64_t i = next.fetch_add(1, std::memory_order_relaxed);
      if (i >= n) return;
      try {
        fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!first) first = std::current_exception();
        next.store(n);
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < workers; ++t) pool.emplace_back(body);
  body();
  for (auto& th : pool) th.join();
  if (first) std::rethrow_exception(first);
}

// ---------------------------------------------------------------- geometry

double norm3(const double* a, const double* b) {
  const double dx = a[0] - b[0];
  const double dy = a[1] - b[1];
  const double dz = a[2] - b[2];
  const double s = dx * dx + dy * dy;  // no contraction (-ffp-contract=off)
  return std::sqrt(s + dz * dz);
}

// model.cpp:45-52, generalised to a (tx, rx) pair.
double sensed_range(double scale, const double* tx, const double* rx,
                    const double* x) {
  const double d_tx = norm3(x, tx);
  const double d_rx = norm3(x, rx);
  if (d_tx == 0.0 || d_rx == 0.0)
    throw domain_error_t("degenerate geometry: target coincides with a station");
  return scale * (d_tx + d_rx);
}

// model.cpp:108-111: origin + spacing * (k mod nx, k div nx), x fastest.
void grid_point(const or_grid& g, int64_t k, double* out) {
  const int64_t nx = g.n[0], ny = g.n[1];
  const int64_t ix = k % nx;
  const int64_t iy = (k / nx) % ny;
  const int64_t iz = k / (nx * ny);
  const double p0 = g.spacing[0] * static_cast<double>(ix);
  const double p1 = g.spacing[1] * static_cast<double>(iy);
  const double p2 = g.spacing[2] * static_cast<double>(iz);
  out[0] = g.origin[0] + p0;
  out[1] = g.origin[1] + p1;
  out[2] = g.origin[2] + p2;
}

int64_t grid_size(const or_grid& g) {
  return static_cast<int64_t>(g.n[0]) * g.n[1] * g.n[2];
}

void check_wave(const or_wave& w) {
  if (w.n_samples < 2) throw std::invalid_argument("waveform: n_samples must be >= 2");
  if (w.os_range < 1) throw std::invalid_argument("hop table: oversampling must be >= 1");
  if (!(w.range_scale > 0.0)) throw std::invalid_argument("waveform: bandwidth must be positive");
  if (w.n_pairs < 1) throw std::invalid_argument("geometry: at least one TX-RX pair required");
}

// ---------------------------------------------------------------- rng

uint64_t splitmix64(uint64_t x) {  // rng.hpp:11-16
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

uint64_t substream(uint64_t seed, uint64_t a, uint64_t b) {  // rng.hpp:20-25
  uint64_t x = splitmix64(seed ^ 0x6a09e667f3bcc909ull);
  x = splitmix64(x + 0x9e3779b97f4a7c15ull * (a + 1));
  x = splitmix64(x + 0xbf58476d1ce4e5b9ull * (b + 1));
  return x;
}

// Counter-addressable replacement for Rng::uniform (rng.hpp:31-34): draw c of
// the SplitMix64 stream seeded with `key`, 53-bit mantissa in [0, 1).
double uniform(uint64_t key, uint64_t c) {
  const uint64_t v = splitmix64(key + 0x9e3779b97f4a7c15ull * c);
  return static_cast<double>(v >> 11) * 0x1.0p-53;
}

// Rng::complex_gaussian (rng.hpp:42-48) on two counter draws.
cplx complex_gaussian(double sigma, double u1, double u2) {
  const double amp = sigma * std::sqrt(-std::log1p(-u1));
  const double ph = 6.283185307179586 * u2;
  return {amp * std::cos(ph), amp * std::sin(ph)};
}

struct Scene {
  std::vector<double> tgt;    // [K][3]
  std::vector<cplx> alpha;    // [K][P]
  std::vector<double> sigma;  // [P]
};

// sample_scene (montecarlo.cpp:48-66) + BASELINE extensions. Draw layout of
// the scene substream (seed, trial, kSceneTag):
//   [0, K*D)            target positions, D = dims
//   [K*D, K*D + 2KP)    amplitude draws, 2 per (target, pair)
//   [.., + P)           per-pair SNR draws (snr_mode 1)
Scene sample_scene(const or_wave& w, const or_campaign& c, uint64_t trial) {
  const int K = c.n_targets, P = w.n_pairs, D = c.dims;
  if (K < 1) throw std::invalid_argument("campaign: n_targets must be >= 1");
  if (D != 2 && D != 3) throw std::invalid_argument("campaign: dims must be 2 or 3");
  const uint64_t key = substream(c.seed, trial, kSceneTag);
  Scene s;
  s.tgt.assign(static_cast<size_t>(K) * 3, 0.0);
  for (int k = 0; k < K; ++k)
    for (int d = 0; d < 3; ++d) {
      double v = c.area_lo[d];
      if (d < D) {
        const double u = uniform(key, static_cast<uint64_t>(k * D + d));
        v = c.area_lo[d] + (c.area_hi[d] - c.area_lo[d]) * u;
      }
      s.tgt[static_cast<size_t>(k) * 3 + d] = v;
    }
  const uint64_t amp0 = static_cast<uint64_t>(K) * D;
  s.alpha.assign(static_cast<size_t>(K) * P, cplx(0.0, 0.0));
  for (int k = 0; k < K; ++k)
    for (int p = 0; p < P; ++p) {
      const bool shared = (c.amp_mode == 0 || c.amp_mode == 2);
      const int pp = shared ? 0 : p;
      const uint64_t at = amp0 + 2ull * (static_cast<uint64_t>(k) * P + pp);
      const double u0 = uniform(key, at), u1 = uniform(key, at + 1);
      cplx a;
      if (c.amp_mode == 0 || c.amp_mode == 1) {
        a = std::polar(1.0, kTwoPi * u0);
      } else if (c.amp_mode == 2 || c.amp_mode == 3) {
        a = complex_gaussian(1.0, u0, u1);
      } else {
        throw std::invalid_argument("campaign: unknown amp_mode");
      }
      s.alpha[static_cast<size_t>(k) * P + p] = a;
    }
  const uint64_t snr0 = amp0 + 2ull * K * P;
  s.sigma.assign(static_cast<size_t>(P), 0.0);
  for (int p = 0; p < P; ++p) {
    double sig;
    if (c.snr_mode == 0) {
      sig = std::pow(10.0, -c.snr_db / 20.0);  // synth.cpp:10-13, alpha_ref 1
    } else if (c.snr_mode == 1) {
      const double u = uniform(key, snr0 + p);
      const double snr = c.snr_lo + (c.snr_hi - c.snr_lo) * u;
      sig = std::pow(10.0, -snr / 20.0);
    } else if (c.snr_mode == 2) {
      sig = 0.0;
    } else {
      throw std::invalid_argument("campaign: unknown snr_mode");
    }
    s.sigma[static_cast<size_t>(p)] = sig;
  }
  return s;
}

// synthesize_frame + add_noise (synth.cpp:15-49) for one trial, Mc = 1:
//   y_p[n] = sum_k alpha_kp exp(j 2pi r_p(x_k) n / N) + w_p[n]
// noise substream (seed, trial, p), draws (2n, 2n+1) per sample.
void synth_trial(const or_wave& w, const or_campaign& c, uint64_t trial,
                 int wrap, double* out /*[P][N][2]*/, double* truth) {
  const Scene s = sample_scene(w, c, trial);
  const int P = w.n_pairs, N = w.n_samples, K = c.n_targets;
  std::vector<cplx> y(static_cast<size_t>(N));
  for (int p = 0; p < P; ++p) {
    std::fill(y.begin(), y.end(), cplx(0.0, 0.0));
    for (int k = 0; k < K; ++k) {
      const double r = sensed_range(w.range_scale, w.tx + 3 * p, w.rx + 3 * p,
                                    &s.tgt[static_cast<size_t>(k) * 3]);
      if (!wrap && !(r >= 0.0 && r < static_cast<double>(N)))
        throw std::runtime_error("scene outside unambiguous window");
      const double step = kTwoPi * r / static_cast<double>(N);  // model.cpp:71-77
      const cplx a = s.alpha[static_cast<size_t>(k) * P + p];
      for (int n = 0; n < N; ++n)
        y[static_cast<size_t>(n)] += a * std::polar(1.0, step * static_cast<double>(n));
    }
    const double sig = s.sigma[static_cast<size_t>(p)];
    if (sig != 0.0) {
      const uint64_t key = substream(c.seed, trial, static_cast<uint64_t>(p));
      for (int n = 0; n < N; ++n)
        y[static_cast<size_t>(n)] += complex_gaussian(
            sig, uniform(key, 2ull * n), uniform(key, 2ull * n + 1));
    }
    double* o = out + static_cast<size_t>(p) * N * 2;
    for (int n = 0; n < N; ++n) {
      o[2 * n] = y[static_cast<size_t>(n)].real();
      o[2 * n + 1] = y[static_cast<size_t>(n)].imag();
    }
  }
  if (truth)
    for (int i = 0; i < 3 * K; ++i) truth[i] = s.tgt[static_cast<size_t>(i)];
}

// ---------------------------------------------------------------- fft

// Forward, unnormalised, zero-padded DFT of one row (fft.hpp:7-10,
// fft.cpp:132-146): out[k] = sum_s in[s] exp(-j 2pi k s / m). Iterative
// radix-2 for power-of-two m, literal DFT otherwise.
void dft_row(const double* in, int n, int m, cplx* out,
             const std::vector<cplx>& tw) {
  for (int k = 0; k < m; ++k) out[k] = 0.0;
  const bool pow2 = (m & (m - 1)) == 0;
  if (!pow2) {
    for (int k = 0; k < m; ++k) {
      cplx s(0.0, 0.0);
      for (int t = 0; t < n; ++t) {
        const int64_t e = (static_cast<int64_t>(k) * t) % m;
        s += cplx(in[2 * t], in[2 * t + 1]) * tw[static_cast<size_t>(e)];
      }
      out[k] = s;
    }
    return;
  }
  int bits = 0;
  while ((1 << bits) < m) ++bits;
  for (int t = 0; t < n; ++t) {
    unsigned r = 0;
    for (int b = 0; b < bits; ++b)
      if (t & (1 << b)) r |= 1u << (bits - 1 - b);
    out[r] = cplx(in[2 * t], in[2 * t + 1]);
  }
  for (int len = 2; len <= m; len <<= 1) {
    const int half = len >> 1;
    const int stride = m / len;
    for (int i = 0; i < m; i += len)
      for (int j = 0; j < half; ++j) {
        const cplx u = out[i + j];
        const cplx v = out[i + j + half] * tw[static_cast<size_t>(j) * stride];
        out[i + j] = u + v;
        out[i + j + half] = u - v;
      }
  }
}

std::vector<cplx> twiddles(int m) {
  std::vector<cplx> tw(static_cast<size_t>(m));
  for (int k = 0; k < m; ++k) {
    const double a = -kTwoPi * static_cast<double>(k) / static_cast<double>(m);
    tw[static_cast<size_t>(k)] = cplx(std::cos(a), std::sin(a));
  }
  return tw;
}

// ---------------------------------------------------------------- fit_atom

// interp.cpp:21-37: D(delta) = sum_m exp(j2pi delta m / n), phasor
// recurrence re-seeded every 1024 steps.
cplx atom_kernel(double delta, int n) {
  const double step = kTwoPi * delta / static_cast<double>(n);
  const double wr = std::cos(step), wi = std::sin(step);
  double pr = 1.0, pim = 0.0, re = 0.0, im = 0.0;
  for (int m = 0; m < n; ++m) {
    if ((m & 1023) == 0) {
      pr = std::cos(step * static_cast<double>(m));
      pim = std::sin(step * static_cast<double>(m));
    }
    re += pr;
    im += pim;
    const double nr = pr * wr - pim * wi;
    pim = pr * wi + pim * wr;
    pr = nr;
  }
  return {re, im};
}

double wrap_range(double r, int n) {  // interp.cpp:39-44
  double w = std::fmod(r, static_cast<double>(n));
  if (w < 0.0) w += static_cast<double>(n);
  if (w >= static_cast<double>(n)) w = 0.0;
  return w;
}

// Eigen::LLT lower-triangular unblocked factorisation; false on a
// non-positive pivot (the reference then regularises, interp.cpp:130-144).
bool llt_solve(const cplx g[3][3], const cplx b[3], cplx c[3]) {
  cplx L[3][3] = {};
  for (int k = 0; k < 3; ++k) {
    double x = g[k][k].real();
    for (int j = 0; j < k; ++j) x -= std::norm(L[k][j]);
    if (!(x > 0.0)) return false;
    const double d = std::sqrt(x);
    L[k][k] = d;
    for (int i = k + 1; i < 3; ++i) {
      cplx s = g[i][k];
      for (int j = 0; j < k; ++j) s -= L[i][j] * std::conj(L[k][j]);
      L[i][k] = s / d;
    }
  }
  cplx y[3];
  for (int i = 0; i < 3; ++i) {
    cplx s = b[i];
    for (int j = 0; j < i; ++j) s -= L[i][j] * y[j];
    y[i] = s / L[i][i];
  }
  for (int i = 2; i >= 0; --i) {
    cplx s = y[i];
    for (int j = i + 1; j < 3; ++j) s -= std::conj(L[j][i]) * c[j];
    c[i] = s / L[i][i];
  }
  return true;
}

// full-pivot LU fallback (Eigen fullPivLu().solve)
void lu_solve(const cplx g[3][3], const cplx b[3], cplx c[3]) {
  cplx a[3][4];
  int col[3] = {0, 1, 2};
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) a[i][j] = g[i][j];
    a[i][3] = b[i];
  }
  for (int k = 0; k < 3; ++k) {
    int pi = k, pj = k;
    double best = -1.0;
    for (int i = k; i < 3; ++i)
      for (int j = k; j < 3; ++j)
        if (std::abs(a[i][j]) > best) best = std::abs(a[i][j]), pi = i, pj = j;
    for (int j = 0; j < 4; ++j) std::swap(a[k][j], a[pi][j]);
    for (int i = 0; i < 3; ++i) std::swap(a[i][k], a[i][pj]);
    std::swap(col[k], col[pj]);
    if (best == 0.0) continue;
    for (int i = k + 1; i < 3; ++i) {
      const cplx f = a[i][k] / a[k][k];
      for (int j = k; j < 4; ++j) a[i][j] -= f * a[k][j];
    }
  }
  cplx x[3];
  for (int i = 2; i >= 0; --i) {
    cplx s = a[i][3];
    for (int j = i + 1; j < 3; ++j) s -= a[i][j] * x[j];
    x[i] = (a[i][i] == cplx(0.0, 0.0)) ? cplx(0.0, 0.0) : s / a[i][i];
  }
  for (int i = 0; i < 3; ++i) c[col[i]] = x[i];
}

int scheme_order(int s) {
  switch (s) {
    case OR_NEAREST: return 1;
    case OR_LINEAR: return 2;
    case OR_POLY3: return 3;
    case OR_POLAR: return 3;
  }
  throw std::invalid_argument("unknown interpolation scheme");
}

struct Fit {
  int k = 0;
  uint32_t idx[3] = {0, 0, 0};
  cplx c[3];
  double residual = 0.0;
};

// fit_atom (interp.cpp:78-154) + the polar scheme:
// nearest / linear / poly3 restated; polar uses the same (i-1, i, i+1)
// triple with real circular-arc weights (Ekanadham et al. 2011 polar
// interpolation, anchors one FFT-grid step apart).
Fit fit_atom(int n_samples, int os, double r, int scheme) {
  if (n_samples < 2 || os < 1) throw std::invalid_argument("fit_atom: bad sizes");
  const int n_fft = n_samples * os;
  const double rw = wrap_range(r, n_samples);
  const double pos = rw * static_cast<double>(os);
  Fit f;
  f.k = scheme_order(scheme);
  switch (scheme) {
    case OR_NEAREST: {
      const long i = static_cast<long>(std::llround(pos)) % n_fft;
      f.idx[0] = static_cast<uint32_t>(i);
      f.c[0] = 1.0;
      break;
    }
    case OR_LINEAR: {
      const long i0 = static_cast<long>(std::floor(pos));
      const double t = pos - static_cast<double>(i0);
      f.idx[0] = static_cast<uint32_t>(i0 % n_fft);
      f.idx[1] = static_cast<uint32_t>((i0 + 1) % n_fft);
      f.c[0] = 1.0 - t;
      f.c[1] = t;
      break;
    }
    case OR_POLY3:
    case OR_POLAR: {
      const long i = static_cast<long>(std::llround(pos));
      f.idx[0] = static_cast<uint32_t>((i - 1 + n_fft) % n_fft);
      f.idx[1] = static_cast<uint32_t>(i % n_fft);
      f.idx[2] = static_cast<uint32_t>((i + 1) % n_fft);
      break;
    }
  }
  double rbar[3] = {0.0, 0.0, 0.0};
  for (int j = 0; j < f.k; ++j)
    rbar[j] = static_cast<double>(f.idx[j]) / static_cast<double>(os);
  cplx gram[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
  cplx rhs[3] = {0.0, 0.0, 0.0};
  for (int j = 0; j < f.k; ++j) {
    rhs[j] = atom_kernel(rbar[j] - rw, n_samples);
    for (int l = 0; l < f.k; ++l) gram[j][l] = atom_kernel(rbar[j] - rbar[l], n_samples);
  }
  if (scheme == OR_POLY3) {
    cplx c[3];
    if (!llt_solve(gram, rhs, c)) {
      cplx g2[3][3];
      const double tr = gram[0][0].real() + gram[1][1].real() + gram[2][2].real();
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) g2[a][b] = gram[a][b];
      for (int a = 0; a < 3; ++a) g2[a][a] += 1e-12 * tr;
      if (!llt_solve(g2, rhs, c)) lu_solve(g2, rhs, c);
    }
    for (int j = 0; j < 3; ++j) f.c[j] = c[j];
  } else if (scheme == OR_POLAR) {
    // anchors f- = a(rbar0), f0 = a(rbar1), f+ = a(rbar2), one grid step h
    // apart; circle through them: chord |f0 - f+| = 2 rho sin(theta/2),
    // |f+ - f-| = 2 rho sin(theta)  =>  cos(theta/2) = d2 / (2 d1).
    const double nn = static_cast<double>(n_samples);
    const double h = 1.0 / static_cast<double>(os);
    const double d1 = std::sqrt(std::max(0.0, 2.0 * nn - 2.0 * atom_kernel(h, n_samples).real()));
    const double d2 = std::sqrt(std::max(0.0, 2.0 * nn - 2.0 * atom_kernel(2.0 * h, n_samples).real()));
    double half = d2 / (2.0 * d1);
    half = std::min(1.0, std::max(-1.0, half));
    const double theta = 2.0 * std::acos(half);
    const double t = pos - static_cast<double>(std::llround(pos));  // in steps, [-.5,.5]
    const double ct = std::cos(theta * t), st = std::sin(theta * t);
    const double one_m_c = 1.0 - std::cos(theta);
    const double a = (1.0 - ct) / one_m_c;
    const double b = st / (2.0 * std::sin(theta));
    f.c[0] = 0.5 * a - b;
    f.c[1] = 1.0 - a;
    f.c[2] = 0.5 * a + b;
  }
  // residual^2 = n - 2 Re(c^H b) + c^H G c   (interp.cpp:146-152)
  cplx quad(0.0, 0.0), cross(0.0, 0.0);
  for (int j = 0; j < f.k; ++j) {
    cplx gc(0.0, 0.0);
    for (int l = 0; l < f.k; ++l) gc += gram[j][l] * f.c[l];
    quad += std::conj(f.c[j]) * gc;
    cross += std::conj(f.c[j]) * rhs[j];
  }
  f.residual = std::sqrt(std::max(0.0, static_cast<double>(n_samples) -
                                           2.0 * cross.real() + quad.real()));
  return f;
}

// hop_bin_value (hopping.cpp:59-102) with Mc = 1 for one trial, all bins.
void hop_map_trial(const cplx* spec /*[P][M]*/, int P, int M,
                   const uint32_t* idx, const double* coef, int64_t G, int K,
                   int magnitude, double* map) {
  for (int64_t b = 0; b < G; ++b) {
    double value = 0.0;
    for (int p = 0; p < P; ++p) {
      const size_t at = (static_cast<size_t>(b) * P + p) * K;
      const cplx* z = spec + static_cast<size_t>(p) * M;
      double vr = 0.0, vi = 0.0;
      for (int j = 0; j < K; ++j) {
        const double cr = coef[2 * (at + j)], ci = coef[2 * (at + j) + 1];
        const cplx zz = z[idx[at + j]];
        if (j == 0) {
          vr = cr * zz.real() - ci * zz.imag();
          vi = cr * zz.imag() + ci * zz.real();
        } else {
          vr = vr + cr * zz.real() - ci * zz.imag();
          vi = vi + cr * zz.imag() + ci * zz.real();
        }
      }
      const double pw = vr * vr + vi * vi;
      value += magnitude ? std::sqrt(pw) : pw;
    }
    map[b] = value;
  }
}

// conj_atom (direct.cpp:20-35)
void conj_atom(double r, int n, double* cre, double* cim) {
  const double step = -kTwoPi * r / static_cast<double>(n);
  const double wr = std::cos(step), wi = std::sin(step);
  double pr = 1.0, pi = 0.0;
  for (int m = 0; m < n; ++m) {
    if ((m & 1023) == 0) {
      pr = std::cos(step * static_cast<double>(m));
      pi = std::sin(step * static_cast<double>(m));
    }
    cre[m] = pr;
    cim[m] = pi;
    const double nr = pr * wr - pi * wi;
    pi = pr * wi + pi * wr;
    pr = nr;
  }
}

// location_decision_map (direct.cpp:90-144) for one trial, Mc = 1, 256-bin
// chunks; the four real GEMM terms accumulate as tr = re*cr - im*ci,
// ti = re*ci + im*cr.
void direct_map_trial(const double* frame /*[P][N][2]*/, const or_wave& w,
                      const or_grid& g, int magnitude, double* map,
                      std::vector<double>& cre, std::vector<double>& cim) {
  const int P = w.n_pairs, N = w.n_samples;
  const int64_t G = grid_size(g);
  cre.resize(static_cast<size_t>(N));
  cim.resize(static_cast<size_t>(N));
  for (int64_t b = 0; b < G; ++b) map[b] = 0.0;
  double x[3];
  for (int64_t b = 0; b < G; ++b) {
    grid_point(g, b, x);
    double acc = 0.0;
    for (int p = 0; p < P; ++p) {
      const double r = sensed_range(w.range_scale, w.tx + 3 * p, w.rx + 3 * p, x);
      conj_atom(r, N, cre.data(), cim.data());
      const double* y = frame + static_cast<size_t>(p) * N * 2;
      double rr = 0.0, ii = 0.0, ri = 0.0, ir = 0.0;
      for (int s = 0; s < N; ++s) {
        rr += y[2 * s] * cre[static_cast<size_t>(s)];
        ii += y[2 * s + 1] * cim[static_cast<size_t>(s)];
        ri += y[2 * s] * cim[static_cast<size_t>(s)];
        ir += y[2 * s + 1] * cre[static_cast<size_t>(s)];
      }
      const double tr = rr - ii;
      const double ti = ri + ir;
      const double pw = tr * tr + ti * ti;
      acc += magnitude ? std::sqrt(pw) : pw;
    }
    map[b] = acc;
  }
}

int64_t argmax(const double* v, int64_t n) {  // direct.cpp:55-62
  if (n <= 0) throw std::invalid_argument("argmax of empty scan");
  int64_t best = 0;
  for (int64_t i = 1; i < n; ++i)
    if (v[i] > v[best]) best = i;
  return best;
}

}  // namespace

extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }
uint64_t or_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t or_substream(uint64_t s, uint64_t a, uint64_t b) { return substream(s, a, b); }
double or_uniform(uint64_t key, uint64_t c) { return uniform(key, c); }

double or_sensed_range(double scale, const double* tx, const double* rx,
                       const double* x, int* status) {
  double r = 0.0;
  const int st = guarded([&] { r = sensed_range(scale, tx, rx, x); });
  if (status) *status = st;
  return r;
}

void or_grid_point(const or_grid* g, int64_t k, double* out3) { grid_point(*g, k, out3); }

int or_scheme_order(int scheme) {
  int k = 0;
  if (guarded([&] { k = scheme_order(scheme); }) != 0) return -1;
  return k;
}

int or_fit_atom(int n_samples, int os, double r, int scheme, uint32_t* idx3,
                double* coef6, double* residual) {
  return guarded([&] {
    const Fit f = fit_atom(n_samples, os, r, scheme);
    for (int j = 0; j < 3; ++j) {
      idx3[j] = f.idx[j];
      coef6[2 * j] = f.c[j].real();
      coef6[2 * j + 1] = f.c[j].imag();
    }
    if (residual) *residual = f.residual;
  });
}

// precompute_hop_table (interp.cpp:156-223): window check naming up to 8
// offenders, then per-bin fits; layout [bin][pair][K].
int or_build_table(const or_wave* w, const or_grid* g, int scheme, int wrap,
                   int n_threads, uint32_t* idx, double* coef, double* max_residual) {
  return guarded([&] {
    check_wave(*w);
    const int K = scheme_order(scheme);
    const int64_t G = grid_size(*g);
    if (G <= 0) throw std::invalid_argument("hop table: empty grid");
    const int P = w->n_pairs;
    double x[3];
    if (!wrap) {
      std::string offenders;
      int64_t count = 0;
      for (int64_t b = 0; b < G; ++b) {
        grid_point(*g, b, x);
        for (int p = 0; p < P; ++p) {
          const double r = sensed_range(w->range_scale, w->tx + 3 * p, w->rx + 3 * p, x);
          if (r >= 0.0 && r < static_cast<double>(w->n_samples)) continue;
          ++count;
          if (count <= 8) {
            char buf[64];
            std::snprintf(buf, sizeof buf, "%s(bin %lld, rx %d)",
                          offenders.empty() ? "" : ", ", static_cast<long long>(b), p);
            offenders += buf;
          }
        }
      }
      if (count > 0) {
        if (count > 8) offenders += ", ...";
        throw std::runtime_error(
            "hop table: sensed range outside [0, n_samples) at " +
            std::to_string(count) + " grid entries: " + offenders);
      }
    }
    std::vector<double> worst(static_cast<size_t>(G), 0.0);
    parallel_for(G, n_threads, [&](int64_t b) {
      double xb[3];
      grid_point(*g, b, xb);
      double wst = 0.0;
      for (int p = 0; p < P; ++p) {
        const double r = sensed_range(w->range_scale, w->tx + 3 * p, w->rx + 3 * p, xb);
        const Fit f = fit_atom(w->n_samples, w->os_range, r, scheme);
        const size_t at = (static_cast<size_t>(b) * P + p) * K;
        for (int j = 0; j < K; ++j) {
          idx[at + j] = f.idx[j];
          coef[2 * (at + j)] = f.c[j].real();
          coef[2 * (at + j) + 1] = f.c[j].imag();
        }
        wst = std::max(wst, f.residual);
      }
      worst[static_cast<size_t>(b)] = wst;
    });
    double mr = 0.0;
    for (double v : worst) mr = std::max(mr, v);
    if (max_residual) *max_residual = mr;
  });
}

int or_table_rows(const or_wave* w, const or_grid* g, int scheme, const int64_t* bins,
                  int64_t n, int n_threads, uint32_t* idx, double* coef) {
  return guarded([&] {
    check_wave(*w);
    const int K = scheme_order(scheme);
    const int64_t G = grid_size(*g);
    const int P = w->n_pairs;
    for (int64_t i = 0; i < n; ++i)
      if (bins[i] < 0 || bins[i] >= G) throw std::invalid_argument("table rows: bin out of range");
    parallel_for(n, n_threads, [&](int64_t i) {
      const int64_t b = bins[i];
      double xb[3];
      grid_point(*g, b, xb);
      for (int p = 0; p < P; ++p) {
        const double r = sensed_range(w->range_scale, w->tx + 3 * p, w->rx + 3 * p, xb);
        const Fit f = fit_atom(w->n_samples, w->os_range, r, scheme);
        const size_t at = (static_cast<size_t>(i) * P + p) * K;
        for (int j = 0; j < K; ++j) {
          idx[at + j] = f.idx[j];
          coef[2 * (at + j)] = f.c[j].real();
          coef[2 * (at + j) + 1] = f.c[j].imag();
        }
      }
    });
  });
}

int or_hop_map_onfly(const double* spectra, int32_t n_trials, const or_wave* w,
                     const or_grid* g, int scheme, int magnitude, int n_threads, double* map) {
  return guarded([&] {
    check_wave(*w);
    const int K = scheme_order(scheme);
    const int64_t G = grid_size(*g);
    const int P = w->n_pairs, M = w->n_samples * w->os_range;
    const auto* sp = reinterpret_cast<const cplx*>(spectra);
    constexpr int64_t kChunk = 1024;  // hopping.cpp:15
    parallel_for((G + kChunk - 1) / kChunk, n_threads, [&](int64_t ch) {
      std::vector<uint32_t> idx(static_cast<size_t>(P) * K);
      std::vector<double> coef(static_cast<size_t>(P) * K * 2);
      const int64_t b1 = std::min(G, (ch + 1) * kChunk);
      for (int64_t b = ch * kChunk; b < b1; ++b) {
        double xb[3];
        grid_point(*g, b, xb);
        for (int p = 0; p < P; ++p) {
          const double r = sensed_range(w->range_scale, w->tx + 3 * p, w->rx + 3 * p, xb);
          const Fit f = fit_atom(w->n_samples, w->os_range, r, scheme);
          for (int j = 0; j < K; ++j) {
            idx[static_cast<size_t>(p) * K + j] = f.idx[j];
            coef[2 * (static_cast<size_t>(p) * K + j)] = f.c[j].real();
            coef[2 * (static_cast<size_t>(p) * K + j) + 1] = f.c[j].imag();
          }
        }
        for (int32_t t = 0; t < n_trials; ++t)  // one bin of each trial's map
          hop_map_trial(sp + static_cast<size_t>(t) * P * M, P, M, idx.data(), coef.data(), 1, K,
                        magnitude, map + static_cast<size_t>(t) * G + b);
      }
    });
  });
}

int or_scene_sample(const or_wave* w, const or_campaign* c, uint64_t trial,
                    double* targets, double* alpha, double* sigma) {
  return guarded([&] {
    const Scene s = sample_scene(*w, *c, trial);
    for (size_t i = 0; i < s.tgt.size(); ++i) targets[i] = s.tgt[i];
    for (size_t i = 0; i < s.alpha.size(); ++i) {
      alpha[2 * i] = s.alpha[i].real();
      alpha[2 * i + 1] = s.alpha[i].imag();
    }
    for (size_t i = 0; i < s.sigma.size(); ++i) sigma[i] = s.sigma[i];
  });
}

int or_synth(const or_wave* w, const or_campaign* c, uint64_t trial0,
             int32_t n_trials, int wrap, double* frames, double* truth) {
  return guarded([&] {
    check_wave(*w);
    const size_t per = static_cast<size_t>(w->n_pairs) * w->n_samples * 2;
    for (int32_t t = 0; t < n_trials; ++t)
      synth_trial(*w, *c, trial0 + static_cast<uint64_t>(t), wrap, frames + per * t,
                  truth ? truth + static_cast<size_t>(t) * c->n_targets * 3 : nullptr);
  });
}

int or_spectra(const double* frames, int64_t rows, int32_t n, int32_t m, double* out) {
  return guarded([&] {
    if (m < n) throw std::invalid_argument("fft: output shorter than input");
    const std::vector<cplx> tw = twiddles(m);
    std::vector<cplx> buf(static_cast<size_t>(m));
    for (int64_t r = 0; r < rows; ++r) {
      dft_row(frames + static_cast<size_t>(r) * n * 2, n, m, buf.data(), tw);
      double* o = out + static_cast<size_t>(r) * m * 2;
      for (int k = 0; k < m; ++k) {
        o[2 * k] = buf[static_cast<size_t>(k)].real();
        o[2 * k + 1] = buf[static_cast<size_t>(k)].imag();
      }
    }
  });
}

int or_hop_map(const double* spectra, int32_t n_trials, int32_t n_pairs, int32_t m,
               const uint32_t* idx, const double* coef, int64_t n_bins, int32_t k,
               int magnitude, double* map) {
  return guarded([&] {
    if (k < 1 || k > 3) throw std::invalid_argument("hop: unsupported interpolation order");
    const size_t per = static_cast<size_t>(n_pairs) * m;
    for (int32_t t = 0; t < n_trials; ++t)
      hop_map_trial(reinterpret_cast<const cplx*>(spectra) + per * t, n_pairs, m, idx,
                    coef, n_bins, k, magnitude, map + static_cast<size_t>(n_bins) * t);
  });
}

// scan_planes / hop_bin_value over Mc chirps (hopping.cpp:59-117): the
// reference's slow-time axis, value(bin) = sum_q sum_mc |sum_j c_j Z_q(mc, I_j)|^2
// (pairs outer, chirps inner). spectra [T][P][Mc][M][2], power combine.
int or_hop_map_mc(const double* spectra, int32_t n_trials, int32_t n_pairs, int32_t n_chirps,
                  int32_t m, const uint32_t* idx, const double* coef, int64_t n_bins, int32_t k,
                  double* map) {
  return guarded([&] {
    if (k < 1 || k > 3) throw std::invalid_argument("hop: unsupported interpolation order");
    const auto* sp = reinterpret_cast<const cplx*>(spectra);
    for (int32_t t = 0; t < n_trials; ++t)
      for (int64_t b = 0; b < n_bins; ++b) {
        double value = 0.0;
        for (int p = 0; p < n_pairs; ++p) {
          const size_t at = (static_cast<size_t>(b) * n_pairs + p) * k;
          for (int mc = 0; mc < n_chirps; ++mc) {
            const cplx* z = sp + ((static_cast<size_t>(t) * n_pairs + p) * n_chirps + mc) * m;
            double vr = 0.0, vi = 0.0;
            for (int j = 0; j < k; ++j) {
              const double cr = coef[2 * (at + j)], ci = coef[2 * (at + j) + 1];
              const cplx zz = z[idx[at + j]];
              vr = vr + cr * zz.real() - ci * zz.imag();
              vi = vi + cr * zz.imag() + ci * zz.real();
            }
            value += vr * vr + vi * vi;
          }
        }
        map[static_cast<size_t>(t) * n_bins + b] = value;
      }
  });
}

int or_direct_map(const double* frames, int32_t n_trials, const or_wave* w,
                  const or_grid* g, int magnitude, int n_threads, double* map) {
  return guarded([&] {
    check_wave(*w);
    const int64_t G = grid_size(*g);
    if (G <= 0) throw std::invalid_argument("decision: empty grid");
    const size_t per = static_cast<size_t>(w->n_pairs) * w->n_samples * 2;
    parallel_for(n_trials, n_threads, [&](int64_t t) {
      std::vector<double> cre, cim;
      direct_map_trial(frames + per * t, *w, *g, magnitude, map + static_cast<size_t>(G) * t,
                       cre, cim);
    });
  });
}

// Indirect pipeline, location stage (src/indirect.cpp:10-83) at Mc = 1:
// range_doppler_map of one receiver's frame is the modulus of its
// zero-padded range spectrum (n_d = os_doppler * 1 rows; os_doppler = 1), its
// peak() the first maximum in row-major order, r_hat = col / os_range
// (indirect.cpp:27-29, 41-56). spectra [rows][m][2] (or_spectra's layout).
int or_range_peaks(const double* spectra, int64_t rows, int32_t m, int32_t os_range,
                   double* rhat) {
  return guarded([&] {
    if (os_range < 1) throw std::invalid_argument("range_doppler_map: oversampling must be >= 1");
    for (int64_t r = 0; r < rows; ++r) {
      const double* z = spectra + 2 * static_cast<size_t>(m) * r;
      double best = -1.0;
      int32_t col = 0;
      for (int32_t k = 0; k < m; ++k) {
        const double v = std::sqrt(z[2 * k] * z[2 * k] + z[2 * k + 1] * z[2 * k + 1]);
        if (v > best) {
          best = v;
          col = k;
        }
      }
      rhat[r] = static_cast<double>(col) / static_cast<double>(os_range);
    }
  });
}

// multilaterate_location (indirect.cpp:58-83): argmin over the grid of
// sum_q (sensed_range(x) - r_hat_q)^2, q ascending, first minimum wins.
// rhat [T][P]; idx [T]; residual [T].
int or_multilaterate(const or_wave* w, const or_grid* g, const double* rhat, int32_t n_trials,
                     int n_threads, int64_t* idx, double* residual) {
  return guarded([&] {
    check_wave(*w);
    const int64_t G = grid_size(*g);
    if (G <= 0) throw std::invalid_argument("multilateration: empty grid");
    const int P = w->n_pairs;
    std::vector<double> r(static_cast<size_t>(G) * P);
    for (int64_t b = 0; b < G; ++b) {
      double x[3];
      grid_point(*g, b, x);
      for (int p = 0; p < P; ++p)
        r[static_cast<size_t>(b) * P + p] =
            sensed_range(w->range_scale, w->tx + 3 * p, w->rx + 3 * p, x);
    }
    parallel_for(n_trials, n_threads, [&](int64_t t) {
      const double* rh = rhat + static_cast<size_t>(t) * P;
      double best = -1.0;
      int64_t bi = 0;
      for (int64_t b = 0; b < G; ++b) {
        double res = 0.0;
        for (int p = 0; p < P; ++p) {
          const double d = r[static_cast<size_t>(b) * P + p] - rh[p];
          res += d * d;
        }
        if (best < 0.0 || res < best) {
          best = res;
          bi = b;
        }
      }
      idx[t] = bi;
      residual[t] = best;
    });
  });
}

// ---------------------------------------------------------------- velocity
// VelocityGrid (model.hpp:93-107, model.cpp:116-131): point k =
// spacing * (k % n - half, k / n - half), n = 2 half + 1 (2-D, z = 0).
static void velocity_point(double spacing, int half, int64_t k, double* v) {
  const int64_t n = 2 * static_cast<int64_t>(half) + 1;
  v[0] = spacing * static_cast<double>(k % n - half);
  v[1] = spacing * static_cast<double>(k / n - half);
  v[2] = 0.0;
}

// doppler_scale * (unit(x - tx) + unit(x - rx)): the slow-time bins per m/s
// of velocity along each axis (sensed_doppler, model.cpp:54-64)
static void doppler_dirs(const double* tx, const double* rx, const double* x, double scale,
                         double* dir) {
  const double ftx[3] = {x[0] - tx[0], x[1] - tx[1], x[2] - tx[2]};
  const double frx[3] = {x[0] - rx[0], x[1] - rx[1], x[2] - rx[2]};
  const double dtx = std::sqrt(ftx[0] * ftx[0] + ftx[1] * ftx[1] + ftx[2] * ftx[2]);
  const double drx = std::sqrt(frx[0] * frx[0] + frx[1] * frx[1] + frx[2] * frx[2]);
  if (dtx == 0.0 || drx == 0.0)
    throw std::domain_error("degenerate geometry: target coincides with a station");
  for (int d = 0; d < 3; ++d) dir[d] = scale * (ftx[d] / dtx + frx[d] / drx);
}

static double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// hop_velocity (hopping.cpp:185-236), batched over trials at their located
// bins: per pair, exact range compression at x_hat with conj(range_atom),
// the zero-padded slow-time DFT (n_d = os_d * Mc) and its power; then the
// velocity-grid scan of nearest Doppler bins (lround, modulo n_d), first
// maximum. frames [T][P][Mc][N][2].
int or_hop_velocity(const double* frames, int32_t n_trials, int32_t n_chirps, const or_wave* w,
                    const or_grid* g, double doppler_scale, double spacing, int32_t half,
                    int32_t os_d, const int64_t* loc, int64_t* vidx, double* vval) {
  return guarded([&] {
    check_wave(*w);
    if (os_d < 1) throw std::invalid_argument("hop velocity: oversampling must be >= 1");
    if (half < 0) throw std::invalid_argument("hop velocity: empty grid");
    const int P = w->n_pairs, N = w->n_samples, Mc = n_chirps, nd = os_d * Mc;
    const int64_t V = (2 * static_cast<int64_t>(half) + 1) * (2 * static_cast<int64_t>(half) + 1);
    const std::vector<cplx> tw = twiddles(nd);
    for (int32_t t = 0; t < n_trials; ++t) {
      double x[3];
      grid_point(*g, loc[t], x);
      std::vector<double> power(static_cast<size_t>(P) * nd), dirs(3 * static_cast<size_t>(P));
      std::vector<double> h(2 * static_cast<size_t>(Mc));
      std::vector<cplx> spec(static_cast<size_t>(nd));
      for (int q = 0; q < P; ++q) {
        const double r = sensed_range(w->range_scale, w->tx + 3 * q, w->rx + 3 * q, x);
        const double* y = frames + ((static_cast<size_t>(t) * P + q) * Mc) * N * 2;
        for (int m = 0; m < Mc; ++m) {
          cplx acc(0.0, 0.0);
          for (int n = 0; n < N; ++n) {
            const cplx ca = std::conj(std::polar(1.0, kTwoPi * r / N * static_cast<double>(n)));
            acc += cplx(y[(static_cast<size_t>(m) * N + n) * 2], y[(static_cast<size_t>(m) * N + n) * 2 + 1]) * ca;
          }
          h[2 * m] = acc.real();
          h[2 * m + 1] = acc.imag();
        }
        dft_row(h.data(), Mc, nd, spec.data(), tw);
        for (int i = 0; i < nd; ++i) power[static_cast<size_t>(q) * nd + i] = std::norm(spec[static_cast<size_t>(i)]);
        doppler_dirs(w->tx + 3 * q, w->rx + 3 * q, x, doppler_scale, &dirs[3 * static_cast<size_t>(q)]);
      }
      int64_t best = 0;
      double best_value = -1.0;
      for (int64_t k = 0; k < V; ++k) {
        double v[3];
        velocity_point(spacing, half, k, v);
        double value = 0.0;
        for (int q = 0; q < P; ++q) {
          const double u = dot3(&dirs[3 * static_cast<size_t>(q)], v);
          const long bin = std::lround(u * static_cast<double>(os_d));
          const int idx = static_cast<int>(((bin % nd) + nd) % nd);
          value += power[static_cast<size_t>(q) * nd + idx];
        }
        if (value > best_value) {
          best_value = value;
          best = k;
        }
      }
      vidx[t] = best;
      vval[t] = best_value;
    }
  });
}

// direct_velocity (direct.cpp:145-228): range compression with conj_atom,
// then per velocity point sum_q |sum_m h_q[m] conj(b(u_q))[m]|^2, first max.
int or_direct_velocity(const double* frames, int32_t n_trials, int32_t n_chirps, const or_wave* w,
                       const or_grid* g, double doppler_scale, double spacing, int32_t half,
                       const int64_t* loc, int64_t* vidx, double* vval) {
  return guarded([&] {
    check_wave(*w);
    if (half < 0) throw std::invalid_argument("velocity scan: empty grid");
    const int P = w->n_pairs, N = w->n_samples, Mc = n_chirps;
    const int64_t V = (2 * static_cast<int64_t>(half) + 1) * (2 * static_cast<int64_t>(half) + 1);
    std::vector<double> cre(static_cast<size_t>(std::max(N, Mc))), cim(cre.size());
    for (int32_t t = 0; t < n_trials; ++t) {
      double x[3];
      grid_point(*g, loc[t], x);
      std::vector<cplx> h(static_cast<size_t>(P) * Mc);
      std::vector<double> dirs(3 * static_cast<size_t>(P));
      for (int q = 0; q < P; ++q) {
        const double r = sensed_range(w->range_scale, w->tx + 3 * q, w->rx + 3 * q, x);
        conj_atom(r, N, cre.data(), cim.data());
        const double* y = frames + ((static_cast<size_t>(t) * P + q) * Mc) * N * 2;
        for (int m = 0; m < Mc; ++m) {
          cplx acc(0.0, 0.0);
          for (int n = 0; n < N; ++n)
            acc += cplx(y[(static_cast<size_t>(m) * N + n) * 2], y[(static_cast<size_t>(m) * N + n) * 2 + 1]) *
                   cplx(cre[static_cast<size_t>(n)], cim[static_cast<size_t>(n)]);
          h[static_cast<size_t>(q) * Mc + m] = acc;
        }
        doppler_dirs(w->tx + 3 * q, w->rx + 3 * q, x, doppler_scale, &dirs[3 * static_cast<size_t>(q)]);
      }
      int64_t best = 0;
      double best_value = -1.0;
      for (int64_t k = 0; k < V; ++k) {
        double v[3];
        velocity_point(spacing, half, k, v);
        double value = 0.0;
        for (int q = 0; q < P; ++q) {
          conj_atom(dot3(&dirs[3 * static_cast<size_t>(q)], v), Mc, cre.data(), cim.data());
          double zr = 0.0, zi = 0.0;
          for (int m = 0; m < Mc; ++m) {
            const cplx hm = h[static_cast<size_t>(q) * Mc + m];
            zr += hm.real() * cre[static_cast<size_t>(m)] - hm.imag() * cim[static_cast<size_t>(m)];
            zi += hm.real() * cim[static_cast<size_t>(m)] + hm.imag() * cre[static_cast<size_t>(m)];
          }
          value += zr * zr + zi * zi;
        }
        if (value > best_value) {
          best_value = value;
          best = k;
        }
      }
      vidx[t] = best;
      vval[t] = best_value;
    }
  });
}

int64_t or_argmax(const double* v, int64_t n) {
  int64_t r = -1;
  if (guarded([&] { r = argmax(v, n); }) != 0) return -1;
  return r;
}

// Top-K local maxima over the lattice neighbourhood (8 in 2-D, 26 in 3-D).
// A bin qualifies if its value is > every neighbour with a smaller index and
// >= every neighbour with a larger index (plateaus resolve to their smallest
// index, the argmax_index tie rule, direct.cpp:55-62). Candidates are ranked
// by (value desc, index asc); missing slots get index -1.
int or_topk_local_max(const double* map, const or_grid* g, int32_t k,
                      int64_t* idx_out, double* val_out) {
  return guarded([&] {
    const int64_t nx = g->n[0], ny = g->n[1], nz = g->n[2];
    std::vector<std::pair<double, int64_t>> cand;
    for (int64_t z = 0; z < nz; ++z)
      for (int64_t y = 0; y < ny; ++y)
        for (int64_t x = 0; x < nx; ++x) {
          const int64_t i = (z * ny + y) * nx + x;
          const double v = map[i];
          bool ok = true;
          for (int dz = -1; dz <= 1 && ok; ++dz)
            for (int dy = -1; dy <= 1 && ok; ++dy)
              for (int dx = -1; dx <= 1 && ok; ++dx) {
                if (!dx && !dy && !dz) continue;
                const int64_t xx = x + dx, yy = y + dy, zz = z + dz;
                if (xx < 0 || yy < 0 || zz < 0 || xx >= nx || yy >= ny || zz >= nz) continue;
                const int64_t j = (zz * ny + yy) * nx + xx;
                ok = (j < i) ? (v > map[j]) : (v >= map[j]);
              }
          if (ok) cand.emplace_back(v, i);
        }
    std::sort(cand.begin(), cand.end(), [](const auto& a, const auto& b) {
      return a.first > b.first || (a.first == b.first && a.second < b.second);
    });
    for (int32_t j = 0; j < k; ++j) {
      if (static_cast<size_t>(j) < cand.size()) {
        idx_out[j] = cand[static_cast<size_t>(j)].second;
        val_out[j] = cand[static_cast<size_t>(j)].first;
      } else {
        idx_out[j] = -1;
        val_out[j] = 0.0;
      }
    }
  });
}

int or_campaign_hop(const or_wave* w, const or_grid* g, const or_campaign* c,
                    const uint32_t* idx, const double* coef, int32_t k, int magnitude,
                    int wrap, uint64_t trial0, int32_t n_trials, int n_threads,
                    int64_t* est_idx, double* est_val) {
  return guarded([&] {
    check_wave(*w);
    const int P = w->n_pairs, N = w->n_samples, M = N * w->os_range;
    const int64_t G = grid_size(*g);
    const std::vector<cplx> tw = twiddles(M);
    parallel_for(n_trials, n_threads, [&](int64_t t) {
      std::vector<double> frame(static_cast<size_t>(P) * N * 2);
      std::vector<cplx> spec(static_cast<size_t>(P) * M);
      std::vector<double> map(static_cast<size_t>(G));
      synth_trial(*w, *c, trial0 + static_cast<uint64_t>(t), wrap, frame.data(), nullptr);
      for (int p = 0; p < P; ++p)
        dft_row(frame.data() + static_cast<size_t>(p) * N * 2, N, M,
                spec.data() + static_cast<size_t>(p) * M, tw);
      // hop scan in fixed 1024-bin chunks (hopping.cpp:15, 104-117)
      for (int64_t b0 = 0; b0 < G; b0 += 1024) {
        const int64_t nb = std::min<int64_t>(1024, G - b0);
        hop_map_trial(spec.data(), P, M, idx + static_cast<size_t>(b0) * P * k,
                      coef + static_cast<size_t>(b0) * P * k * 2, nb, k, magnitude,
                      map.data() + b0);
      }
      const int64_t best = argmax(map.data(), G);
      est_idx[t] = best;
      est_val[t] = map[static_cast<size_t>(best)];
    });
  });
}

// Top-k local maxima per trial (BASELINE c3/c5 multi-target campaigns): the
// hop pipeline of or_campaign_hop, then or_topk_local_max on each map.
int or_campaign_hop_topk(const or_wave* w, const or_grid* g, const or_campaign* c,
                         const uint32_t* idx, const double* coef, int32_t k, int magnitude,
                         int wrap, uint64_t trial0, int32_t n_trials, int32_t topk,
                         int n_threads, int64_t* est_idx, double* est_val) {
  return guarded([&] {
    check_wave(*w);
    if (topk < 1 || topk > 8) throw std::invalid_argument("top-k: k must be in [1, 8]");
    const int P = w->n_pairs, N = w->n_samples, M = N * w->os_range;
    const int64_t G = grid_size(*g);
    const std::vector<cplx> tw = twiddles(M);
    std::string first_err;
    parallel_for(n_trials, n_threads, [&](int64_t t) {
      std::vector<double> frame(static_cast<size_t>(P) * N * 2);
      std::vector<cplx> spec(static_cast<size_t>(P) * M);
      std::vector<double> map(static_cast<size_t>(G));
      synth_trial(*w, *c, trial0 + static_cast<uint64_t>(t), wrap, frame.data(), nullptr);
      for (int p = 0; p < P; ++p)
        dft_row(frame.data() + static_cast<size_t>(p) * N * 2, N, M,
                spec.data() + static_cast<size_t>(p) * M, tw);
      for (int64_t b0 = 0; b0 < G; b0 += 1024) {
        const int64_t nb = std::min<int64_t>(1024, G - b0);
        hop_map_trial(spec.data(), P, M, idx + static_cast<size_t>(b0) * P * k,
                      coef + static_cast<size_t>(b0) * P * k * 2, nb, k, magnitude,
                      map.data() + b0);
      }
      if (or_topk_local_max(map.data(), g, topk, est_idx + t * topk, est_val + t * topk) != 0)
        throw std::runtime_error(g_err);
    });
  });
}

// Campaign statistics of one batch (run_monte_carlo's hit_ratio,
// montecarlo.cpp:181-190, extended with location RMSE and K-target
// assignment). Per trial, truths x_i (i < kt, rows of truth [T][kt][3]) are
// matched to estimates (est [T][ke] grid bins, -1 = none) by the injective
// assignment of least total squared distance over the permutations of
// max(kt, ke) slots in lexicographic order (first minimum kept); an
// unmatched truth counts at distance `miss_m`. Distances are formed as
// sqrt((dx*dx + dy*dy) + dz*dz), every operation rounded separately.
// out[0] += estimates counted, out[1 + j] += hits within thresholds[j],
// out[1 + nth] += sum of squared distances, out[2 + nth] += hits within
// half_res, out[3 + nth] += sum of distances. assign [T][kt] (nullable):
// the estimate slot matched to each truth (-1 = missed).
int or_trial_stats(const or_grid* g, const int64_t* est, int32_t ke, const double* truth,
                   int32_t kt, int32_t n_trials, const double* thresholds, int32_t nth,
                   double half_res, double miss_m, double* out, int32_t* assign) {
  return guarded([&] {
    const int n = std::max(ke, kt);
    if (n < 1 || n > 6) throw std::invalid_argument("stats: at most 6 targets / estimates");
    std::vector<int> perm(static_cast<size_t>(n)), bestp(static_cast<size_t>(n));
    std::vector<double> dist(static_cast<size_t>(kt) * n);
    for (int32_t t = 0; t < n_trials; ++t) {
      for (int i = 0; i < kt; ++i)
        for (int j = 0; j < n; ++j) {
          const int64_t b = j < ke ? est[static_cast<int64_t>(t) * ke + j] : -1;
          double d = miss_m;
          if (b >= 0) {
            double x[3];
            grid_point(*g, b, x);
            const double* tr = truth + (static_cast<int64_t>(t) * kt + i) * 3;
            const double dx = x[0] - tr[0], dy = x[1] - tr[1], dz = x[2] - tr[2];
            d = std::sqrt((dx * dx + dy * dy) + dz * dz);
          }
          dist[static_cast<size_t>(i) * n + j] = d;
        }
      for (int j = 0; j < n; ++j) perm[static_cast<size_t>(j)] = j;
      double best = 0.0;
      bool have = false;
      do {
        double cost = 0.0;
        for (int i = 0; i < kt; ++i) {
          const double d = dist[static_cast<size_t>(i) * n + perm[static_cast<size_t>(i)]];
          cost = cost + d * d;
        }
        if (!have || cost < best) {
          best = cost;
          bestp = perm;
          have = true;
        }
      } while (std::next_permutation(perm.begin(), perm.end()));
      for (int i = 0; i < kt; ++i) {
        const int j = bestp[static_cast<size_t>(i)];
        const double d = dist[static_cast<size_t>(i) * n + j];
        const bool matched = j < ke && est[static_cast<int64_t>(t) * ke + j] >= 0;
        if (assign) assign[static_cast<int64_t>(t) * kt + i] = matched ? j : -1;
        out[0] += 1.0;
        for (int h = 0; h < nth; ++h)
          if (d <= thresholds[h]) out[1 + h] += 1.0;
        out[1 + nth] += d * d;
        if (d <= half_res) out[2 + nth] += 1.0;
        out[3 + nth] += d;
      }
    }
  });
}

int or_campaign_direct(const or_wave* w, const or_grid* g, const or_campaign* c,
                       int magnitude, int wrap, uint64_t trial0, int32_t n_trials,
                       int n_threads, int64_t* est_idx, double* est_val) {
  return guarded([&] {
    check_wave(*w);
    const int P = w->n_pairs, N = w->n_samples;
    const int64_t G = grid_size(*g);
    parallel_for(n_trials, n_threads, [&](int64_t t) {
      std::vector<double> frame(static_cast<size_t>(P) * N * 2);
      std::vector<double> map(static_cast<size_t>(G));
      std::vector<double> cre, cim;
      synth_trial(*w, *c, trial0 + static_cast<uint64_t>(t), wrap, frame.data(), nullptr);
      direct_map_trial(frame.data(), *w, *g, magnitude, map.data(), cre, cim);
      const int64_t best = argmax(map.data(), G);
      est_idx[t] = best;
      est_val[t] = map[static_cast<size_t>(best)];
    });
  });
}

}  // extern "C"
