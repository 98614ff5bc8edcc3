// gh_table.cu — offline mapping operator on the device (fp64) and the gather
// plan derived from it.
//
// Reference: precompute_hop_table / fit_atom (src/interp.cpp:21-223). The
// index rules (llround / floor on the wrapped position, interp.cpp:88-111)
// only see sensed_range, fmod and one product, all rounded individually here
// (__dmul_rn/__dadd_rn/__dsqrt_rn) exactly as the -ffp-contract=off oracle
// does, so indices are bit-identical; coefficients agree to ~1e-15.
//
// The gather plan turns the [bin][pair][K] operator into what the gather
// kernel streams: per location tile (a 3-D box of bins) and pair, a window of
// range rows [base, base+len) mod M staged in shared memory, and per
// (bin, pair) the uint16 shared-memory row of its first FFT bin.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <unordered_map>

#include "gh_internal.cuh"

namespace gh {
namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;

struct cd {
  double re, im;
};
__device__ inline cd cmul(cd a, cd b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
__device__ inline cd cadd(cd a, cd b) { return {a.re + b.re, a.im + b.im}; }
__device__ inline cd csub(cd a, cd b) { return {a.re - b.re, a.im - b.im}; }
__device__ inline cd cconj(cd a) { return {a.re, -a.im}; }
__device__ inline cd cdivr(cd a, double d) { return {a.re / d, a.im / d}; }
__device__ inline cd cdiv(cd a, cd b) {
  const double den = b.re * b.re + b.im * b.im;
  return {(a.re * b.re + a.im * b.im) / den, (a.im * b.re - a.re * b.im) / den};
}
__device__ inline double cabs2(cd a) { return a.re * a.re + a.im * a.im; }

// interp.cpp:21-37 atom_kernel: phasor recurrence re-seeded every 1024 steps
__device__ cd atom_kernel(double delta, int n) {
  const double step = kTwoPi * delta / (double)n;
  double wi, wr;
  sincos(step, &wi, &wr);
  double pr = 1.0, pim = 0.0, re = 0.0, im = 0.0;
  for (int m = 0; m < n; ++m) {
    if ((m & 1023) == 0) sincos(step * (double)m, &pim, &pr);
    re += pr;
    im += pim;
    const double nr = pr * wr - pim * wi;
    pim = pr * wi + pim * wr;
    pr = nr;
  }
  return {re, im};
}

__device__ double wrap_range(double r, int n) {  // interp.cpp:39-44
  double w = fmod(r, (double)n);
  if (w < 0.0) w = __dadd_rn(w, (double)n);
  if (w >= (double)n) w = 0.0;
  return w;
}

__device__ bool llt_solve(const cd g[3][3], const cd b[3], cd c[3]) {
  cd L[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) L[i][j] = {0.0, 0.0};
  for (int k = 0; k < 3; ++k) {
    double x = g[k][k].re;
    for (int j = 0; j < k; ++j) x -= cabs2(L[k][j]);
    if (!(x > 0.0)) return false;
    const double d = sqrt(x);
    L[k][k] = {d, 0.0};
    for (int i = k + 1; i < 3; ++i) {
      cd s = g[i][k];
      for (int j = 0; j < k; ++j) s = csub(s, cmul(L[i][j], cconj(L[k][j])));
      L[i][k] = cdivr(s, d);
    }
  }
  cd y[3];
  for (int i = 0; i < 3; ++i) {
    cd s = b[i];
    for (int j = 0; j < i; ++j) s = csub(s, cmul(L[i][j], y[j]));
    y[i] = cdivr(s, L[i][i].re);
  }
  for (int i = 2; i >= 0; --i) {
    cd s = y[i];
    for (int j = i + 1; j < 3; ++j) s = csub(s, cmul(cconj(L[j][i]), c[j]));
    c[i] = cdivr(s, L[i][i].re);
  }
  return true;
}

__device__ void lu_solve(const cd g[3][3], const cd b[3], cd c[3]) {
  cd a[3][4];
  int col[3] = {0, 1, 2};
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) a[i][j] = g[i][j];
    a[i][3] = b[i];
  }
  for (int k = 0; k < 3; ++k) {
    int pi = k, pj = k;
    double best = -1.0;
    for (int i = k; i < 3; ++i)
      for (int j = k; j < 3; ++j) {
        const double v = sqrt(cabs2(a[i][j]));
        if (v > best) best = v, pi = i, pj = j;
      }
    for (int j = 0; j < 4; ++j) { cd t = a[k][j]; a[k][j] = a[pi][j]; a[pi][j] = t; }
    for (int i = 0; i < 3; ++i) { cd t = a[i][k]; a[i][k] = a[i][pj]; a[i][pj] = t; }
    { int t = col[k]; col[k] = col[pj]; col[pj] = t; }
    if (best == 0.0) continue;
    for (int i = k + 1; i < 3; ++i) {
      const cd f = cdiv(a[i][k], a[k][k]);
      for (int j = k; j < 4; ++j) a[i][j] = csub(a[i][j], cmul(f, a[k][j]));
    }
  }
  cd x[3];
  for (int i = 2; i >= 0; --i) {
    cd s = a[i][3];
    for (int j = i + 1; j < 3; ++j) s = csub(s, cmul(a[i][j], x[j]));
    x[i] = (a[i][i].re == 0.0 && a[i][i].im == 0.0) ? cd{0.0, 0.0} : cdiv(s, a[i][i]);
  }
  for (int i = 0; i < 3; ++i) c[col[i]] = x[i];
}

// fit_atom (interp.cpp:78-154) + polar (oracle/gridhop_oracle.cpp fit_atom)
__device__ double fit_atom(int n_samples, int os, double r, int scheme, uint32_t* idx, cd* c) {
  const int n_fft = n_samples * os;
  const double rw = wrap_range(r, n_samples);
  const double pos = __dmul_rn(rw, (double)os);
  int k = scheme == GH_NEAREST ? 1 : (scheme == GH_LINEAR ? 2 : 3);
  for (int j = 0; j < 3; ++j) { idx[j] = 0; c[j] = {0.0, 0.0}; }
  long long ir = llround(pos);
  if (scheme == GH_NEAREST) {
    idx[0] = (uint32_t)(ir % n_fft);
    c[0] = {1.0, 0.0};
  } else if (scheme == GH_LINEAR) {
    const long long i0 = (long long)floor(pos);
    const double t = __dsub_rn(pos, (double)i0);
    idx[0] = (uint32_t)(i0 % n_fft);
    idx[1] = (uint32_t)((i0 + 1) % n_fft);
    c[0] = {__dsub_rn(1.0, t), 0.0};
    c[1] = {t, 0.0};
  } else {
    idx[0] = (uint32_t)((ir - 1 + n_fft) % n_fft);
    idx[1] = (uint32_t)(ir % n_fft);
    idx[2] = (uint32_t)((ir + 1) % n_fft);
  }
  double rbar[3] = {0.0, 0.0, 0.0};
  for (int j = 0; j < k; ++j) rbar[j] = (double)idx[j] / (double)os;
  cd gram[3][3], rhs[3];
  for (int a = 0; a < 3; ++a) {
    rhs[a] = {0.0, 0.0};
    for (int b = 0; b < 3; ++b) gram[a][b] = {a == b ? 1.0 : 0.0, 0.0};
  }
  for (int j = 0; j < k; ++j) {
    rhs[j] = atom_kernel(rbar[j] - rw, n_samples);
    for (int l = 0; l < k; ++l) gram[j][l] = atom_kernel(rbar[j] - rbar[l], n_samples);
  }
  if (scheme == GH_POLY3) {
    if (!llt_solve(gram, rhs, c)) {
      cd g2[3][3];
      const double tr = gram[0][0].re + gram[1][1].re + gram[2][2].re;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) g2[a][b] = gram[a][b];
      for (int a = 0; a < 3; ++a) g2[a][a].re += 1e-12 * tr;
      if (!llt_solve(g2, rhs, c)) lu_solve(g2, rhs, c);
    }
  } else if (scheme == GH_POLAR) {
    const double nn = (double)n_samples;
    const double h = 1.0 / (double)os;
    const double d1 = sqrt(fmax(0.0, 2.0 * nn - 2.0 * atom_kernel(h, n_samples).re));
    const double d2 = sqrt(fmax(0.0, 2.0 * nn - 2.0 * atom_kernel(2.0 * h, n_samples).re));
    double half = d2 / (2.0 * d1);
    half = fmin(1.0, fmax(-1.0, half));
    const double theta = 2.0 * acos(half);
    const double t = pos - (double)ir;
    const double ct = cos(theta * t), st = sin(theta * t);
    const double a = (1.0 - ct) / (1.0 - cos(theta));
    const double b = st / (2.0 * sin(theta));
    c[0] = {0.5 * a - b, 0.0};
    c[1] = {1.0 - a, 0.0};
    c[2] = {0.5 * a + b, 0.0};
  }
  cd quad = {0.0, 0.0}, cross = {0.0, 0.0};
  for (int j = 0; j < k; ++j) {
    cd gc = {0.0, 0.0};
    for (int l = 0; l < k; ++l) gc = cadd(gc, cmul(gram[j][l], c[l]));
    quad = cadd(quad, cmul(cconj(c[j]), gc));
    cross = cadd(cross, cmul(cconj(c[j]), rhs[j]));
  }
  return sqrt(fmax(0.0, (double)n_samples - 2.0 * cross.re + quad.re));
}

struct BuildArgs {
  gh_grid grid;
  const double* txrx;  // [P][6]
  double scale;
  int P, N, os, K, scheme, wrap;
  int64_t G, bin0;     // local bins, global index of the first
  uint32_t* idx;
  double2* coef;
  uint8_t* flags;      // window (1) / degenerate (2) per entry
  unsigned long long* max_res_bits;
  unsigned long long* n_flag;
};

__global__ void k_build(BuildArgs a) {
  const int64_t total = a.G * a.P;
  double worst = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / a.P;
    const int p = (int)(e % a.P);
    double x[3];
    dgrid_point(a.grid, a.bin0 + b, x);
    const double* tx = a.txrx + 6 * p;
    const double dtx = dnorm3(tx, x[0], x[1], x[2]);
    const double drx = dnorm3(tx + 3, x[0], x[1], x[2]);
    uint8_t fl = 0;
    if (dtx == 0.0 || drx == 0.0) fl |= 2;
    const double r = __dmul_rn(a.scale, __dadd_rn(dtx, drx));
    if (!a.wrap && !(r >= 0.0 && r < (double)a.N)) fl |= 1;
    a.flags[e] = fl;
    if (fl) atomicAdd(a.n_flag, 1ull);
    uint32_t idx[3];
    cd c[3];
    const double res = fit_atom(a.N, a.os, r, a.scheme, idx, c);
    for (int j = 0; j < a.K; ++j) {
      a.idx[e * a.K + j] = idx[j];
      if (a.coef) a.coef[e * a.K + j] = make_double2(c[j].re, c[j].im);
    }
    worst = fmax(worst, res);
  }
  // residuals are >= 0: their IEEE bits order like the values
  for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
  if ((threadIdx.x & 31) == 0)
    atomicMax(a.max_res_bits, (unsigned long long)__double_as_longlong(worst));
}

// fit_atom for caller-chosen ranges (the reference's public fit_atom,
// interp.hpp:41): one thread per range, the table builder's device code
__global__ void k_fit_atoms(int n_samples, int os, const double* r, int n, int scheme,
                           uint32_t* idx, double2* coef, double* res) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t ix[3] = {0u, 0u, 0u};
  cd c[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  res[i] = fit_atom(n_samples, os, r[i], scheme, ix, c);
  for (int j = 0; j < 3; ++j) {
    idx[3 * i + j] = ix[j];
    coef[3 * i + j] = make_double2(c[j].re, c[j].im);
  }
}

// top-K plans: each entry's position in its tile's values plane
// ((ly + 1) * pitch + lx + 1, inside the -inf ring), bit 15 set for halo bins,
// so the gather stores and tracks core maxima without decoding the blocked
// entry order (2-D tiles)
__global__ void k_fill_pos(const TileDesc* tiles, uint16_t* pos) {
  const TileDesc td = tiles[blockIdx.x];
  const int nb = td.wx * td.wy * td.wz, pitch = topk_pitch(td.wx);
  for (int lb = threadIdx.x; lb < nb; lb += blockDim.x) {
    int64_t lx, ly, lz;
    tile_local(td, lb, &lx, &ly, &lz);
    const bool halo = lx < td.cx0 || lx >= td.cx0 + td.cwx || ly < td.cy0 || ly >= td.cy0 + td.cwy;
    pos[td.entry_off + lb] =
        static_cast<uint16_t>(((ly + 1) * pitch + lx + 1) | (halo ? 0x8000 : 0));
  }
}

// smallest flagged entry index strictly above `after` (offender report)
__global__ void k_next_flag(const uint8_t* flags, int64_t total, int64_t after,
                            unsigned long long* out) {
  for (int64_t e = after + 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    if (flags[e]) {
      atomicMin(out, (unsigned long long)e);
      return;
    }
}

// ---------------------------------------------------------------- plan

__device__ inline void tile_bin(const TileDesc& td, const gh_grid& g, int64_t lb, int64_t* gb) {
  int64_t lx, ly, lz;
  tile_local(td, lb, &lx, &ly, &lz);
  *gb = (td.x0 + lx) + (int64_t)g.n[0] * ((td.y0 + ly) + (int64_t)g.n[1] * (td.z0 + lz));
}

// per (tile, pair): floor(min u), ceil(max u), u = r * os unwrapped
__global__ void k_tile_minmax(const TileDesc* tiles, gh_grid g, const double* txrx, double scale,
                              int os, int P, int2* out) {
  const TileDesc td = tiles[blockIdx.x];
  const int64_t nb = (int64_t)td.wx * td.wy * td.wz;
  __shared__ int smin[32], smax[32];
  for (int p = 0; p < P; ++p) {
    int lo = 0x7fffffff, hi = -0x7fffffff;
    const double* tx = txrx + 6 * p;
    for (int64_t lb = threadIdx.x; lb < nb; lb += blockDim.x) {
      int64_t gb;
      tile_bin(td, g, lb, &gb);
      double x[3];
      dgrid_point(g, gb, x);
      const double u = scale * (dnorm3(tx, x[0], x[1], x[2]) + dnorm3(tx + 3, x[0], x[1], x[2])) * os;
      lo = min(lo, (int)floor(u));
      hi = max(hi, (int)ceil(u));
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
      smin[threadIdx.x >> 5] = lo;
      smax[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
        lo = min(lo, smin[w]);
        hi = max(hi, smax[w]);
      }
      out[(int64_t)blockIdx.x * P + p] = make_int2(lo, hi);
    }
    __syncthreads();
  }
}

struct FillArgs {
  const TileDesc* tiles;  // null for the full plan
  gh_grid grid;
  const int4* win;        // [tiles][P] (full: [P])
  const uint32_t* idx;    // [G][P][K]
  const double2* coef;
  int P, K, M, p4, k3, lanes;
  int64_t G, bin0;        // local bins; tiles carry global coordinates
  int64_t n_entries;      // plan entries: row words are stored [p / 4][entry]
  uint16_t* rows;
  float2* coef3;
  float4* coefr;  // real weights (polar): [P][entries]
  int* err;
};

// one CTA per tile (tiled) or grid-stride over bins (full)
__global__ void k_fill_plan(FillArgs a) {
  int64_t entry0 = 0, nb = a.G;
  TileDesc td{};
  const int4* win = a.win;
  if (a.tiles) {
    td = a.tiles[blockIdx.x];
    entry0 = td.entry_off;
    nb = (int64_t)td.wx * td.wy * td.wz;
    win = a.win + (int64_t)blockIdx.x * a.P;
  }
  const int64_t total = nb * a.P;
  const int64_t start = a.tiles ? threadIdx.x : blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t step = a.tiles ? blockDim.x : (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = start; e < total; e += step) {
    const int64_t lb = e / a.P;
    const int p = (int)(e % a.P);
    int64_t gb = entry0 + lb;  // local bin
    if (a.tiles) {
      tile_bin(td, a.grid, lb, &gb);  // global bin
      gb -= a.bin0;
    }
    const int4 w = win[p];
    const int64_t at = (gb * a.P + p) * a.K;
    const int first = (int)a.idx[at];
    const int local = ((first - w.x) % a.M + a.M) % a.M;
    if (local + (a.k3 ? 2 : 0) >= w.y) atomicOr(a.err, 1);
    // stored in 16-byte units of the staged row layout (row * L), so the
    // gather forms the shared-memory address with one shift-add
    const int off16 = (w.z + local) * a.lanes;
    if (off16 > 65535) atomicOr(a.err, 2);
    // word-major ([pair / 4][entry] of 4 x uint16): the gather's lanes load
    // one word of consecutive entries, i.e. contiguous 8-byte runs
    a.rows[((int64_t)(p >> 2) * a.n_entries + entry0 + lb) * 4 + (p & 3)] = (uint16_t)off16;
    if (a.k3 && a.coefr) {
      // polar weights are real (the anchors' chords): 3 floats + pad, one
      // 16-byte load per (bin, pair) in the gather, [pair][entry]
      float w[3];
      for (int j = 0; j < 3; ++j) {
        w[j] = j < a.K ? (float)a.coef[at + j].x : 0.0f;
        if (j < a.K && a.coef[at + j].y != 0.0) atomicOr(a.err, 4);
      }
      a.coefr[(int64_t)p * a.n_entries + entry0 + lb] = make_float4(w[0], w[1], w[2], 0.0f);
    } else if (a.k3) {
      // word-major like the rows: [pair][j][entry]
      for (int j = 0; j < 3; ++j) {
        const double2 c = j < a.K ? a.coef[at + j] : make_double2(0.0, 0.0);
        a.coef3[((int64_t)p * 3 + j) * a.n_entries + entry0 + lb] =
            make_float2((float)c.x, (float)c.y);
      }
    }
  }
}

constexpr size_t kStageBudget = 216 * 1024;  // full-ring plan: one CTA per SM
constexpr size_t kTileBudget = 216 * 1024;   // tiled plans: one CTA per SM

// Bank-conflict-aware bin order for the 16-trial full-ring power plan. A row
// there is 64 bytes (half a shared-memory wavefront) and the gather serves
// two bins per quarter-warp with one LDS.128 per pair: the two rows collide
// when their row indices have equal parity. Bins are re-ordered so that
// entries (2k, 2k+1) have complementary parity vectors over the pairs;
// `binid` maps entries back to bins, which keeps reported indices exact, and
// the order is built so that the smallest-bin tie rule of argmax_index
// (src/direct.cpp:55-62) survives it (see the two cases below).
void permute_for_banks(Ctx* ctx, Table* t, Plan& pl) {
  const int P = t->P, p4 = pl.p4, L = pl.tb * pl.esize / 16;
  const int64_t n = pl.n_entries;
  std::vector<uint16_t> rows(static_cast<size_t>(n) * p4), wm(rows.size());
  GH_CUDA(cudaMemcpyAsync(wm.data(), pl.rows_d, sizeof(uint16_t) * wm.size(),
                          cudaMemcpyDeviceToHost, ctx->stream));
  GH_CUDA(cudaStreamSynchronize(ctx->stream));
  // device layout is word-major [p / 4][entry][p % 4]; work entry-major here
  auto wm_at = [n](int64_t e, int p) {
    return static_cast<size_t>((((int64_t)(p >> 2)) * n + e) * 4 + (p & 3));
  };
  for (int64_t e = 0; e < n; ++e)
    for (int p = 0; p < p4; ++p) rows[static_cast<size_t>(e) * p4 + p] = wm[wm_at(e, p)];
  const unsigned full = (1u << P) - 1u;
  // Bins whose rows equal an earlier bin's for every pair always tie with
  // it and can never win the argmax: they go last (ascending), so entry
  // order still resolves every forced tie to the smallest bin and the
  // gather keeps its branch-free "first strict maximum" update.
  std::vector<uint32_t> uniq, dups;
  {
    std::unordered_map<uint64_t, uint32_t> seen;
    seen.reserve(static_cast<size_t>(n) * 2);
    for (int64_t e = 0; e < n; ++e) {
      uint64_t h = 0;
      for (int p = 0; p < p4; ++p) h = (h << 16) ^ rows[e * p4 + p] ^ (h >> 48);
      bool dup = false;
      auto it = seen.find(h);
      if (it != seen.end())
        dup = std::memcmp(&rows[e * p4], &rows[static_cast<size_t>(it->second) * p4],
                          sizeof(uint16_t) * p4) == 0;
      else
        seen.emplace(h, static_cast<uint32_t>(e));
      (dup ? dups : uniq).push_back(static_cast<uint32_t>(e));
    }
  }
  std::vector<uint32_t> order;
  order.reserve(static_cast<size_t>(n));
  const int64_t nu = static_cast<int64_t>(uniq.size());
  auto parity = [&](uint32_t e) {
    unsigned v = 0;
    for (int p = 0; p < P; ++p) v |= ((rows[static_cast<size_t>(e) * p4 + p] / L) & 1u) << p;
    return v;
  };
  std::vector<std::vector<uint32_t>> bucket(static_cast<size_t>(full) + 1);
  if (P <= 3) {
    // Ordered plan (order_lane_monotone, gh_internal.cuh): every entry pair
    // bank-complementary, every lane group's bins in increasing order, the
    // unmatched bins as an ascending tail from tie_from on.
    std::vector<unsigned> par(static_cast<size_t>(nu));
    for (int64_t u = 0; u < nu; ++u) par[static_cast<size_t>(u)] = parity(uniq[static_cast<size_t>(u)]);
    pl.tie_from = order_lane_monotone(uniq, par, P, &order);
  } else {
    // more couples than entry pairs: greedy matching of v with ~v inside
    // windows of 1024 bins; no lane order, so the gather compares bins on
    // every exact tie (tie_from = 0)
    constexpr int64_t W = 1024;  // even: pairs stay on even entry offsets
    pl.tie_from = 0;
    for (int64_t w0 = 0; w0 < nu; w0 += W) {
      const int64_t w1 = std::min<int64_t>(nu, w0 + W);
      for (auto& b : bucket) b.clear();
      for (int64_t u = w1 - 1; u >= w0; --u) {  // reversed: pop_back yields ascending
        const uint32_t e = uniq[static_cast<size_t>(u)];
        bucket[parity(e)].push_back(e);
      }
      std::vector<uint32_t> rest;
      for (unsigned v = 0; v <= full; ++v) {
        auto& a = bucket[v];
        auto& b = bucket[full ^ v];
        if (v > (full ^ v)) continue;  // each complementary couple once
        while (!a.empty() && !b.empty() && (&a != &b || a.size() >= 2)) {
          order.push_back(a.back());
          a.pop_back();
          order.push_back(b.back());
          b.pop_back();
        }
      }
      for (auto& b : bucket)
        for (auto it = b.rbegin(); it != b.rend(); ++it) rest.push_back(*it);
      std::sort(rest.begin(), rest.end());
      order.insert(order.end(), rest.begin(), rest.end());
    }
  }
  order.insert(order.end(), dups.begin(), dups.end());
  std::vector<uint16_t> prow(rows.size());
  std::vector<uint32_t> binid(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t e = order[static_cast<size_t>(i)];
    std::memcpy(&prow[static_cast<size_t>(i) * p4], &rows[static_cast<size_t>(e) * p4],
                sizeof(uint16_t) * p4);
    binid[static_cast<size_t>(i)] = static_cast<uint32_t>(t->bin0 + e);
  }
  for (int64_t e = 0; e < n; ++e)
    for (int p = 0; p < p4; ++p) wm[wm_at(e, p)] = prow[static_cast<size_t>(e) * p4 + p];
  GH_CUDA(cudaMemcpyAsync(pl.rows_d, wm.data(), sizeof(uint16_t) * wm.size(),
                          cudaMemcpyHostToDevice, ctx->stream));
  GH_CUDA(cudaStreamSynchronize(ctx->stream));  // wm is a host temporary
  GH_CUDA(cudaMalloc(&pl.binid_d, sizeof(uint32_t) * n));
  GH_CUDA(cudaMemcpyAsync(pl.binid_d, binid.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice,
                          ctx->stream));
  // compact rows when every pair's ring row fits one 32-bit word (c1/c2:
  // 3 x 10 bits): the gather then shuffles one word per step, not two
  int bits = 1;
  while ((1 << bits) < t->M) ++bits;
  std::vector<uint32_t> crow;
  if (P * bits <= 32) {
    crow.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      uint32_t w = 0;
      for (int p = 0; p < P; ++p) {
        const uint32_t r = prow[static_cast<size_t>(i) * p4 + p] / L - static_cast<uint32_t>(p * t->M);
        w |= r << (bits * p);
      }
      crow[static_cast<size_t>(i)] = w;
    }
    GH_CUDA(cudaMalloc(&pl.crow_d, sizeof(uint32_t) * n));
    GH_CUDA(cudaMemcpyAsync(pl.crow_d, crow.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice,
                            ctx->stream));
    pl.cbits = bits;
  }
  GH_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace

void build_table_device(Ctx* ctx, Table* t, int wrap) {
  const int64_t total = t->G * t->P;
  GH_CUDA(cudaMalloc(&t->idx_d, sizeof(uint32_t) * total * t->K));
  // nearest (K = 1) coefficients are identically 1: not stored
  if (t->K > 1) GH_CUDA(cudaMalloc(&t->coef_d, sizeof(double2) * total * t->K));
  uint8_t* flags = nullptr;
  unsigned long long* scal = nullptr;  // [0] max residual bits, [1] flag count, [2] next flag
  GH_CUDA(cudaMalloc(&flags, total));
  GH_CUDA(cudaMalloc(&scal, 3 * sizeof(unsigned long long)));
  GH_CUDA(cudaMemsetAsync(scal, 0, 3 * sizeof(unsigned long long), ctx->stream));
  BuildArgs a{};
  a.grid = t->grid;
  a.txrx = t->txrx_d;
  a.scale = t->scale;
  a.P = t->P;
  a.N = t->N;
  a.os = t->os;
  a.K = t->K;
  a.scheme = t->scheme;
  a.wrap = wrap;
  a.G = t->G;
  a.bin0 = t->bin0;
  a.idx = t->idx_d;
  a.coef = t->coef_d;
  a.flags = flags;
  a.max_res_bits = scal;
  a.n_flag = scal + 1;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 127) / 128, 148LL * 64));
  k_build<<<blocks, 128, 0, ctx->stream>>>(a);
  GH_LAUNCHED(ctx);
  unsigned long long h[2];
  GH_CUDA(cudaMemcpyAsync(h, scal, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          ctx->stream));
  GH_CUDA(cudaStreamSynchronize(ctx->stream));
  double mr;
  std::memcpy(&mr, &h[0], sizeof mr);
  t->max_residual = mr;
  std::string err;
  int code = 0;
  if (h[1] > 0) {
    // name up to 8 offenders in (bin, pair) order, interp.cpp:182-201
    std::string names;
    int64_t after = -1;
    bool degenerate = false;
    for (int i = 0; i < 8; ++i) {
      unsigned long long init = ~0ull;
      GH_CUDA(cudaMemcpyAsync(scal + 2, &init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
      k_next_flag<<<blocks, 128, 0, ctx->stream>>>(flags, total, after, scal + 2);
      GH_LAUNCHED(ctx);
      unsigned long long nx;
      GH_CUDA(cudaMemcpyAsync(&nx, scal + 2, sizeof nx, cudaMemcpyDeviceToHost, ctx->stream));
      GH_CUDA(cudaStreamSynchronize(ctx->stream));
      if (nx == ~0ull) break;
      uint8_t fl;
      GH_CUDA(cudaMemcpy(&fl, flags + nx, 1, cudaMemcpyDeviceToHost));
      if (fl & 2) degenerate = true;
      char buf[64];
      std::snprintf(buf, sizeof buf, "%s(bin %lld, rx %d)", names.empty() ? "" : ", ",
                    (long long)(t->bin0 + nx / t->P), (int)(nx % t->P));
      names += buf;
      after = (int64_t)nx;
    }
    if (degenerate) {
      code = GH_EDOMAIN;
      err = "degenerate geometry: target coincides with a station";
    } else {
      if (h[1] > 8) names += ", ...";
      code = GH_ERUNTIME;
      err = "hop table: sensed range outside [0, n_samples) at " + std::to_string(h[1]) +
            " grid entries: " + names;
    }
  }
  cudaFree(flags);
  cudaFree(scal);
  if (code) fail(code, err);
}

Plan& build_plan(Ctx* ctx, Table* t, bool mapmode) {
  Plan& pl = mapmode ? t->plan_map : t->plan;
  if (pl.built) return pl;
  const int P = t->P, M = t->M;
  pl.k3 = t->K > 1;
  pl.esize = pl.k3 ? 8 : 4;
  pl.p4 = (P + 3) / 4 * 4;
  const int ring = pl.k3 ? M + 2 : M;
  // full plan: whole ring per pair, 16 trials per CTA
  const size_t full_bytes = static_cast<size_t>(P) * ring * 16 * pl.esize;
  int* err_d = nullptr;
  GH_CUDA(cudaMalloc(&err_d, sizeof(int)));
  GH_CUDA(cudaMemsetAsync(err_d, 0, sizeof(int), ctx->stream));
  if (full_bytes <= kStageBudget && ring <= 65535 / P) {
    pl.full = true;
    pl.tb = 16;
    pl.n_tiles = 1;
    pl.max_rows = P * ring;
    pl.n_entries = t->G;
    std::vector<int4> win(static_cast<size_t>(P));
    for (int p = 0; p < P; ++p)
      win[static_cast<size_t>(p)] = make_int4(pl.k3 ? M - 1 : 0, ring, p * ring, 0);
    GH_CUDA(cudaMalloc(&pl.win_d, sizeof(int4) * P));
    GH_CUDA(cudaMemcpyAsync(pl.win_d, win.data(), sizeof(int4) * P, cudaMemcpyHostToDevice,
                            ctx->stream));
    GH_CUDA(cudaStreamSynchronize(ctx->stream));
  } else {
    pl.full = false;
    // trial batch: 8 trials of power (32-byte rows) or 16 of complex
    // spectrum (128-byte rows; 8 if that leaves < 40 staged rows per pair).
    // Narrow power rows cost some bank conflicts but buy wider tiles, i.e.
    // fewer staged rows per bin: measured against 16 / 32 trials on c3
    // (15.2 vs 16.2 / 19.3 ms per 4096 trials) and c5 (2x); complex rows
    // measured best at 16 (c4: 25.5 vs 37.9 ms at 8)
    pl.tb = pl.k3 ? 16 : 8;
    while (pl.tb > 8 &&
           static_cast<int>(kTileBudget / (static_cast<size_t>(pl.tb) * pl.esize)) / P < 40)
      pl.tb >>= 1;
    // pair chunks with their own shared-memory regions for the pipelined
    // gather (17-64 pairs: 16 pairs = 4 row-table words per chunk); one
    // chunk otherwise
    pl.chunk_pairs = pl.p4 > 16 ? 16 : pl.p4;
    // 8-trial power rows (32 bytes): entries in 8-bin blocks (tile_local)
    // (argmax plans only: map-mode gathers store each trial's bins
    // contiguously along x, which the plain order keeps)
    const bool blocked = !mapmode && !pl.k3 && pl.tb == 8;
    const bool grid3 = t->grid.n[2] > 1;
    const int bext[3] = {2, grid3 ? 1 : 4, grid3 ? 4 : 1};  // 8-bin block extents
    const int blk_code = 1 + 1 + ((grid3 ? 0 : 2) << 2) + ((grid3 ? 2 : 0) << 4);
    const int n_chunks = (P + pl.chunk_pairs - 1) / pl.chunk_pairs;
    const int budget_rows = static_cast<int>(kTileBudget / (static_cast<size_t>(pl.tb) * pl.esize));
    const int allow = budget_rows / P - 5;
    if (allow < 4) fail(GH_EINVAL, "gather plan: too many pairs for one shared-memory window");
    const gh_grid& g = t->grid;
    const int dims = g.n[2] > 1 ? 3 : 2;
    const double grad = 2.0 * t->scale * t->os;  // max |du/dx| per metre
    double side = allow / (grad * std::sqrt((double)dims));
    struct Tiling {
      std::vector<TileDesc> tiles;
      std::vector<int4> win;
      int max_rows = 0;
      int64_t entries = 0;
    };
    int2* mm_d = nullptr;
    size_t mm_cap = 0;
    TileDesc* scratch_tiles = nullptr;
    size_t tiles_cap = 0;
    // tile boxes of about `side` metres; windows measured on the device
    auto try_tiling = [&](double s) {
      Tiling tl;
      int w[3];
      for (int d = 0; d < 3; ++d) {
        w[d] = g.n[d] > 1 ? std::max(1, (int)std::floor(s / g.spacing[d])) : 1;
        w[d] = std::min(w[d], g.n[d]);
      }
      if (dims == 2) w[2] = 1;
      if (blocked)  // whole blocks (edge tiles may still be ragged)
        for (int d = 0; d < 3; ++d)
          if (w[d] >= bext[d]) w[d] -= w[d] % bext[d];
      // the shard's box: layers [slab_lo, slab_hi) of z (3-D) or y (2-D)
      const int z_lo = dims == 3 ? t->slab_lo : 0, z_hi = dims == 3 ? t->slab_hi : g.n[2];
      const int y_lo = dims == 3 ? 0 : t->slab_lo, y_hi = dims == 3 ? g.n[1] : t->slab_hi;
      int64_t off = 0;
      for (int z = z_lo; z < z_hi; z += w[2])
        for (int y = y_lo; y < y_hi; y += w[1])
          for (int x = 0; x < g.n[0]; x += w[0]) {
            TileDesc td{};
            td.x0 = x;
            td.y0 = y;
            td.z0 = z;
            td.wx = std::min(w[0], g.n[0] - x);
            td.wy = std::min(w[1], y_hi - y);
            td.wz = std::min(w[2], z_hi - z);
            td.entry_off = off;
            td.blk = blocked && td.wx % bext[0] == 0 && td.wy % bext[1] == 0 &&
                             td.wz % bext[2] == 0
                         ? blk_code
                         : 0;
            td.cwx = td.wx;
            td.cwy = td.wy;
            td.cwz = td.wz;
            off += (int64_t)td.wx * td.wy * td.wz;
            tl.tiles.push_back(td);
          }
      tl.entries = off;
      const size_t nt = tl.tiles.size();
      if (nt > tiles_cap) {
        if (scratch_tiles) cudaFree(scratch_tiles);
        GH_CUDA(cudaMalloc(&scratch_tiles, sizeof(TileDesc) * nt));
        tiles_cap = nt;
      }
      if (nt * P > mm_cap) {
        if (mm_d) cudaFree(mm_d);
        GH_CUDA(cudaMalloc(&mm_d, sizeof(int2) * nt * P));
        mm_cap = nt * P;
      }
      GH_CUDA(cudaMemcpyAsync(scratch_tiles, tl.tiles.data(), sizeof(TileDesc) * nt,
                              cudaMemcpyHostToDevice, ctx->stream));
      k_tile_minmax<<<static_cast<int>(nt), 256, 0, ctx->stream>>>(scratch_tiles, g, t->txrx_d,
                                                                   t->scale, t->os, P, mm_d);
      GH_LAUNCHED(ctx);
      std::vector<int2> mm(nt * P);
      GH_CUDA(cudaMemcpyAsync(mm.data(), mm_d, sizeof(int2) * mm.size(), cudaMemcpyDeviceToHost,
                              ctx->stream));
      GH_CUDA(cudaStreamSynchronize(ctx->stream));
      tl.win.assign(mm.size(), make_int4(0, 0, 0, 0));
      // pair chunks own fixed shared-memory regions (the largest chunk
      // window over all tiles), so the gather can restage chunk c of its
      // next item while it still reads the other chunks of this one
      std::vector<int> region(static_cast<size_t>(n_chunks), 0);
      for (size_t ti = 0; ti < nt; ++ti) {
        int rs = 0;
        for (int p = 0; p < P; ++p) {
          const int2 m = mm[ti * P + p];
          int base = m.x - 2, len = m.y - m.x + 5;
          if (len >= ring) {
            base = pl.k3 ? M - 1 : 0;
            len = ring;
          }
          base = ((base % M) + M) % M;
          tl.win[ti * P + p] = make_int4(base, len, 0, 0);
          rs += len;
          if (p % pl.chunk_pairs == pl.chunk_pairs - 1 || p == P - 1) {
            int& r = region[static_cast<size_t>(p / pl.chunk_pairs)];
            r = std::max(r, rs);
            rs = 0;
          }
        }
      }
      std::vector<int> region_off(static_cast<size_t>(n_chunks), 0);
      for (int c = 1; c < n_chunks; ++c)
        region_off[static_cast<size_t>(c)] = region_off[c - 1] + region[c - 1];
      tl.max_rows = region_off.back() + region.back();
      for (size_t ti = 0; ti < nt; ++ti) {
        int rs = 0;
        for (int p = 0; p < P; ++p) {
          if (p % pl.chunk_pairs == 0) rs = region_off[static_cast<size_t>(p / pl.chunk_pairs)];
          tl.win[ti * P + p].z = rs;
          rs += tl.win[ti * P + p].y;
        }
        tl.tiles[ti].rows = rs;
      }
      return tl;
    };
    auto fits = [&](const Tiling& tl) {
      return tl.max_rows <= budget_rows && tl.max_rows <= 65535;
    };
    Tiling best = try_tiling(side);
    for (int i = 0; i < 16 && !fits(best); ++i) {
      side *= 0.75;
      best = try_tiling(side);
    }
    if (!fits(best)) fail(GH_EINVAL, "gather plan: no tiling fits the shared-memory budget");
    // the gradient bound is a worst case: grow while the windows still fit
    for (int i = 0; i < 8 && best.max_rows * 10 < budget_rows * 7; ++i) {
      if (best.tiles.size() <= 1) break;
      side *= 1.25;
      Tiling bigger = try_tiling(side);
      if (!fits(bigger)) break;
      best = std::move(bigger);
    }
    if (scratch_tiles) cudaFree(scratch_tiles);
    if (mm_d) cudaFree(mm_d);
    std::vector<TileDesc>& tiles = best.tiles;
    std::vector<int4>& win = best.win;
    pl.max_rows = best.max_rows;
    pl.n_tiles = static_cast<int>(tiles.size());
    pl.n_entries = best.entries;
    TileDesc* tiles_d = nullptr;
    GH_CUDA(cudaMalloc(&tiles_d, sizeof(TileDesc) * tiles.size()));
    GH_CUDA(cudaMemcpyAsync(tiles_d, tiles.data(), sizeof(TileDesc) * tiles.size(),
                            cudaMemcpyHostToDevice, ctx->stream));
    GH_CUDA(cudaMalloc(&pl.win_d, sizeof(int4) * win.size()));
    GH_CUDA(cudaMemcpyAsync(pl.win_d, win.data(), sizeof(int4) * win.size(),
                            cudaMemcpyHostToDevice, ctx->stream));
    pl.tiles_d = tiles_d;
  }
  GH_CUDA(cudaMalloc(&pl.rows_d, sizeof(uint16_t) * pl.n_entries * pl.p4));
  GH_CUDA(cudaMemsetAsync(pl.rows_d, 0, sizeof(uint16_t) * pl.n_entries * pl.p4, ctx->stream));
  const bool real_w = pl.k3 && t->scheme == GH_POLAR;  // polar coefficients are real
  if (real_w) GH_CUDA(cudaMalloc(&pl.coefr_d, sizeof(float4) * pl.n_entries * P));
  else if (pl.k3) GH_CUDA(cudaMalloc(&pl.coef3_d, sizeof(float2) * pl.n_entries * P * 3));
  FillArgs f{};
  f.tiles = pl.full ? nullptr : pl.tiles_d;
  f.grid = t->grid;
  f.win = pl.win_d;
  f.idx = t->idx_d;
  f.coef = t->coef_d;
  f.P = P;
  f.K = t->K;
  f.M = M;
  f.p4 = pl.p4;
  f.k3 = pl.k3;
  f.lanes = pl.tb * pl.esize / 16;
  f.G = t->G;
  f.bin0 = t->bin0;
  f.rows = pl.rows_d;
  f.n_entries = pl.n_entries;
  f.coef3 = pl.coef3_d;
  f.coefr = pl.coefr_d;
  f.err = err_d;
  if (pl.full) {
    const int blocks = static_cast<int>(std::min<int64_t>((t->G * P + 255) / 256, 148LL * 32));
    k_fill_plan<<<blocks, 256, 0, ctx->stream>>>(f);
  } else {
    k_fill_plan<<<pl.n_tiles, 256, 0, ctx->stream>>>(f);
  }
  GH_LAUNCHED(ctx);
  int herr = 0;
  GH_CUDA(cudaMemcpyAsync(&herr, err_d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  GH_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(err_d);
  if (herr & 4) fail(GH_EINVAL, "hop table: polar coefficients must be real");
  if (herr) fail(GH_ERUNTIME, "gather plan: an index fell outside its staged window");
  if (pl.full && !pl.k3 && P <= 8) permute_for_banks(ctx, t, pl);
  pl.built = true;
  return pl;
}


// ---------------------------------------------------------------- top-K plan

// Fused top-K plans (BASELINE c3: 2-D grid, K = 1, many pairs): 8-trial
// batches as the argmax plan, but each tile's core box is grown by a 1-bin
// halo so the gather itself evaluates every neighbour a core bin's
// local-maximum test needs; the tile's values for its 8 trials then stay in
// shared memory next to the range windows (gh_gather_topk.cu k_gather_topk).
// Windows + values must share one CTA's shared memory, so tiles are smaller
// than the argmax plan's (~56 x 56 bins on c3 instead of ~113 x 113).
constexpr size_t kTopkSmem = 224 * 1024;  // windows + values + lists, per SM

Plan* build_plan_topk(Ctx* ctx, Table* t) {
  Plan& pl = t->plan_topk;
  if (pl.built) return &pl;
  if (!t->topk_fused_ok) return nullptr;
  const gh_grid& g = t->grid;
  const int P = t->P, M = t->M;
  const size_t full_bytes = static_cast<size_t>(P) * M * 16 * 4;
  const bool full_ring = full_bytes <= kStageBudget && M <= 65535 / P;
  if (t->K != 1 || g.n[2] > 1 || full_ring || t->bin0 != 0 ||
      t->G != (int64_t)g.n[0] * g.n[1] || P > 64) {
    t->topk_fused_ok = false;
    return nullptr;
  }
  pl.full = false;
  pl.k3 = 0;
  pl.esize = 4;
  pl.tb = 8;
  pl.p4 = (P + 3) / 4 * 4;
  pl.chunk_pairs = pl.p4;
  pl.halo = true;
  struct Tiling {
    std::vector<TileDesc> tiles;
    std::vector<int4> win;
    int max_rows = 0;
    int64_t entries = 0;
    size_t vals = 0;
    int plane = 0;
  };
  int2* mm_d = nullptr;
  TileDesc* tiles_d = nullptr;
  size_t mm_cap = 0, tiles_cap = 0;
  // core widths: x even, y == 2 mod 4, so interior halo boxes (core + 2)
  // are whole 2 x 4 blocks and run in the blocked entry order
  auto try_tiling = [&](int w) {
    Tiling tl;
    const int cw_x = std::max(2, w - w % 2);
    const int cw_y = std::max(2, w - ((w - 2) % 4 + 4) % 4);
    int64_t off = 0;
    for (int y = 0; y < g.n[1]; y += cw_y)
      for (int x = 0; x < g.n[0]; x += cw_x) {
        TileDesc td{};
        const int ex0 = std::max(0, x - 1), ey0 = std::max(0, y - 1);
        const int ex1 = std::min(g.n[0], x + cw_x + 1), ey1 = std::min(g.n[1], y + cw_y + 1);
        td.x0 = ex0;
        td.y0 = ey0;
        td.z0 = 0;
        td.wx = ex1 - ex0;
        td.wy = ey1 - ey0;
        td.wz = 1;
        td.cx0 = x - ex0;
        td.cy0 = y - ey0;
        td.cz0 = 0;
        td.cwx = std::min(cw_x, g.n[0] - x);
        td.cwy = std::min(cw_y, g.n[1] - y);
        td.cwz = 1;
        td.entry_off = off;
        td.blk = td.wx % 2 == 0 && td.wy % 4 == 0 ? 1 + 1 + (2 << 2) : 0;  // 2 x 4 x 1
        off += (int64_t)td.wx * td.wy;
        tl.plane = std::max(tl.plane, topk_pitch(td.wx) * (td.wy + 2));
        tl.tiles.push_back(td);
      }
    tl.entries = off;
    // trial planes 4 mod 8 floats apart: a gather store's two 4-trial lane
    // halves land in opposite bank halves (+8: the filter's last float4 may
    // run past the ring row)
    tl.plane = (tl.plane + 8 + 3) / 8 * 8 + 4;
    tl.vals = (size_t)tl.plane * 8 * sizeof(float);
    const size_t nt = tl.tiles.size();
    if (nt > tiles_cap) {
      if (tiles_d) cudaFree(tiles_d);
      GH_CUDA(cudaMalloc(&tiles_d, sizeof(TileDesc) * nt));
      tiles_cap = nt;
    }
    if (nt * P > mm_cap) {
      if (mm_d) cudaFree(mm_d);
      GH_CUDA(cudaMalloc(&mm_d, sizeof(int2) * nt * P));
      mm_cap = nt * P;
    }
    GH_CUDA(cudaMemcpyAsync(tiles_d, tl.tiles.data(), sizeof(TileDesc) * nt,
                            cudaMemcpyHostToDevice, ctx->stream));
    k_tile_minmax<<<static_cast<int>(nt), 256, 0, ctx->stream>>>(tiles_d, g, t->txrx_d, t->scale,
                                                                 t->os, P, mm_d);
    GH_LAUNCHED(ctx);
    std::vector<int2> mm(nt * P);
    GH_CUDA(cudaMemcpyAsync(mm.data(), mm_d, sizeof(int2) * mm.size(), cudaMemcpyDeviceToHost,
                            ctx->stream));
    GH_CUDA(cudaStreamSynchronize(ctx->stream));
    tl.win.assign(mm.size(), make_int4(0, 0, 0, 0));
    for (size_t ti = 0; ti < nt; ++ti) {
      int rs = 0;
      for (int p = 0; p < P; ++p) {
        const int2 m = mm[ti * P + p];
        int base = m.x - 2, len = m.y - m.x + 5;
        if (len >= M) {
          base = 0;
          len = M;
        }
        base = ((base % M) + M) % M;
        tl.win[ti * P + p] = make_int4(base, len, rs, 0);
        rs += len;
      }
      tl.tiles[ti].rows = rs;
      tl.max_rows = std::max(tl.max_rows, rs);
    }
    return tl;
  };
  auto smem_of = [&](const Tiling& tl) {
    // windows + two values buffers (the pick of one item overlaps the next
    // item's gather) + the kernel's static lists
    return ((size_t)tl.max_rows * 8 * 4 + 127) / 128 * 128 + 2 * ((tl.vals + 127) / 128 * 128) +
           kTopkListBytes;
  };
  auto fits = [&](const Tiling& tl) {
    return smem_of(tl) <= kTopkSmem && tl.max_rows * 2 <= 65535;  // 16-byte units, L = 2
  };
  // start near values ~ 45 % of the budget, then shrink / grow the core
  int w = static_cast<int>(std::sqrt(0.45 * kTopkSmem / 64.0)) - 3;
  w = std::max(4, std::min(w, std::max(g.n[0], g.n[1])));
  Tiling best = try_tiling(w);
  for (int i = 0; i < 40 && !fits(best) && w > 4; ++i) {
    w = std::max(4, w * 9 / 10);
    best = try_tiling(w);
  }
  if (!fits(best)) {
    cudaFree(tiles_d);
    cudaFree(mm_d);
    t->topk_fused_ok = false;
    return nullptr;
  }
  for (int i = 0; i < 32; ++i) {
    if (w >= std::max(g.n[0], g.n[1])) break;
    Tiling bigger = try_tiling(w + 4);
    if (!fits(bigger)) break;
    best = std::move(bigger);
    w += 4;
  }
  cudaFree(mm_d);
  // final tiles (the scratch holds the last tried tiling): upload `best`
  GH_CUDA(cudaMalloc(&pl.tiles_d, sizeof(TileDesc) * best.tiles.size()));
  GH_CUDA(cudaMemcpyAsync(pl.tiles_d, best.tiles.data(), sizeof(TileDesc) * best.tiles.size(),
                          cudaMemcpyHostToDevice, ctx->stream));
  cudaFree(tiles_d);
  GH_CUDA(cudaMalloc(&pl.win_d, sizeof(int4) * best.win.size()));
  GH_CUDA(cudaMemcpyAsync(pl.win_d, best.win.data(), sizeof(int4) * best.win.size(),
                          cudaMemcpyHostToDevice, ctx->stream));
  pl.n_tiles = static_cast<int>(best.tiles.size());
  pl.max_rows = best.max_rows;
  pl.n_entries = best.entries;
  pl.vals_bytes = best.vals;
  pl.topk_plane = best.plane;
  GH_CUDA(cudaMalloc(&pl.rows_d, sizeof(uint16_t) * pl.n_entries * pl.p4));
  GH_CUDA(cudaMemsetAsync(pl.rows_d, 0, sizeof(uint16_t) * pl.n_entries * pl.p4, ctx->stream));
  int* err_d = nullptr;
  GH_CUDA(cudaMalloc(&err_d, sizeof(int)));
  GH_CUDA(cudaMemsetAsync(err_d, 0, sizeof(int), ctx->stream));
  FillArgs f{};
  f.tiles = pl.tiles_d;
  f.grid = g;
  f.win = pl.win_d;
  f.idx = t->idx_d;
  f.coef = t->coef_d;
  f.P = P;
  f.K = 1;
  f.M = M;
  f.p4 = pl.p4;
  f.k3 = 0;
  f.lanes = 2;
  f.G = t->G;
  f.bin0 = 0;
  f.rows = pl.rows_d;
  f.n_entries = pl.n_entries;
  f.coef3 = nullptr;
  f.err = err_d;
  k_fill_plan<<<pl.n_tiles, 256, 0, ctx->stream>>>(f);
  GH_LAUNCHED(ctx);
  if (best.plane >= 0x8000) fail(GH_EINVAL, "gather plan: top-K tile too large");
  GH_CUDA(cudaMalloc(&pl.pos_d, sizeof(uint16_t) * pl.n_entries));
  k_fill_pos<<<pl.n_tiles, 256, 0, ctx->stream>>>(pl.tiles_d, pl.pos_d);
  GH_LAUNCHED(ctx);
  int herr = 0;
  GH_CUDA(cudaMemcpyAsync(&herr, err_d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  GH_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(err_d);
  if (herr) fail(GH_ERUNTIME, "gather plan: an index fell outside its staged window");
  pl.built = true;
  return &pl;
}

void launch_fit_atoms(Ctx* ctx, int n_samples, int os, const double* r_d, int n, int scheme,
                      uint32_t* idx_d, double2* coef_d, double* res_d) {
  k_fit_atoms<<<(n + 127) / 128, 128, 0, ctx->stream>>>(n_samples, os, r_d, n, scheme, idx_d,
                                                        coef_d, res_d);
  GH_LAUNCHED(ctx);
}

}  // namespace gh
