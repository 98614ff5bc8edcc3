// gh_fft.cu — beat-signal synthesis and the zero-padded range FFT (sm_100a).
//
// Reference: fast_time_spectra / fft_rows (src/hopping.cpp:121-129,
// src/fft.cpp:132-146, include/gridhop/fft.hpp:7-10): out[k] =
// sum_n y[n] exp(-j 2pi k n / M), M = os * N, forward and unnormalised.
// Synthesis restates synthesize_frame + add_noise (src/synth.cpp:15-49) and
// sample_scene (src/montecarlo.cpp:48-66) on the counter-based stream shared
// with the oracle.
//
// Zero padding is pruned exactly: with k = os*m + j,
//   X[os*m + j] = sum_{n<N} (y[n] W_M^{jn}) W_N^{mn},
// i.e. os independent N-point FFTs of twiddled copies of the N samples; the
// padded zeros are never touched. Each N-point FFT runs as Stockham
// radix-16/8/4/2 passes: a thread loads R points, twiddles, does the R-point
// DFT in registers and writes back (one shared-memory round trip and two
// barriers per pass; N = 256 is two passes). Shared memory is padded one
// float2 per 16 so the strided Stockham writes are bank-conflict free.
//
// One CTA owns TB trials of one pair (blockIdx = (trial batch, pair)),
// R_ROWS rows at a time. The epilogue writes either the natural [T][P][M]
// complex layout (parity) or the gather layout [batch][pair][M][TB] — one
// contiguous TB-run per range bin — as power, magnitude or complex.
#include <cuda_runtime.h>

#include "gh_internal.cuh"

namespace gh {
namespace {

constexpr int kFftThreads = 512;
constexpr int kMaxTargets = 8;

struct RowSynth {
  double r[kMaxTargets];      // sensed range of target k for this pair
  float2 alpha[kMaxTargets];  // amplitude of target k on this pair
  double sigma;
  uint64_t noise_key;
};

// sample_scene (montecarlo.cpp:48-66) + BASELINE extensions, restricted to
// pair p: identical draw layout to oracle/gridhop_oracle.cpp sample_scene.
__device__ void row_setup(const SynthParams& sp, int P, int p, uint64_t trial,
                          RowSynth& rs, int* err) {
  const gh_campaign& c = sp.camp;
  const int K = c.n_targets, D = c.dims;
  const uint64_t key = substream(c.seed, trial, kSceneTag);
  const double* tx = sp.txrx_d + 6 * p;
  const double* rx = tx + 3;
  for (int k = 0; k < K; ++k) {
    double x[3];
    for (int d = 0; d < 3; ++d) {
      double v = c.area_lo[d];
      if (d < D) {
        const double u = uniform01(key, (uint64_t)(k * D + d));
        v = __dadd_rn(c.area_lo[d], __dmul_rn(__dsub_rn(c.area_hi[d], c.area_lo[d]), u));
      }
      x[d] = v;
    }
    const double dtx = dnorm3(tx, x[0], x[1], x[2]);
    const double drx = dnorm3(rx, x[0], x[1], x[2]);
    if (dtx == 0.0 || drx == 0.0) atomicOr(err, 2);
    const double r = __dmul_rn(sp.scale, __dadd_rn(dtx, drx));
    rs.r[k] = r;
    const bool shared = (c.amp_mode == 0 || c.amp_mode == 2);
    const uint64_t at = (uint64_t)K * D + 2ull * ((uint64_t)k * P + (shared ? 0 : p));
    const double u0 = uniform01(key, at), u1 = uniform01(key, at + 1);
    double s, co;
    if (c.amp_mode == 0 || c.amp_mode == 1) {
      sincospi(2.0 * u0, &s, &co);
      rs.alpha[k] = make_float2((float)co, (float)s);
    } else {
      const double amp = sqrt(-log1p(-u0));
      sincospi(2.0 * u1, &s, &co);
      rs.alpha[k] = make_float2((float)(amp * co), (float)(amp * s));
    }
  }
  double sig = 0.0;
  if (c.snr_mode == 0) {
    sig = pow(10.0, -c.snr_db / 20.0);
  } else if (c.snr_mode == 1) {
    const uint64_t at = (uint64_t)K * D + 2ull * K * P + p;
    const double u = uniform01(key, at);
    sig = pow(10.0, -(c.snr_lo + (c.snr_hi - c.snr_lo) * u) / 20.0);
  }
  rs.sigma = sig;
  rs.noise_key = substream(c.seed, trial, (uint64_t)p);
}

// One beat-signal sample y_p[n] (synth.cpp:15-49): phases reduced in fp64
// (r n / N reaches ~1e5 turns) before an fp32 sincospi.
__device__ __forceinline__ float2 synth_sample(const RowSynth& rs, int K, int n,
                                               double inv_n) {
  float2 y = make_float2(0.f, 0.f);
  for (int k = 0; k < K; ++k) {
    const double tt = rs.r[k] * (double)n * inv_n;
    const double fr = tt - floor(tt);
    float s, c;
    sincospif((float)(2.0 * fr), &s, &c);
    const float2 a = rs.alpha[k];
    y.x += a.x * c - a.y * s;
    y.y += a.x * s + a.y * c;
  }
  if (rs.sigma != 0.0) {
    const double u1 = uniform01(rs.noise_key, 2ull * n);
    const double u2 = uniform01(rs.noise_key, 2ull * n + 1);
    const float amp = (float)(rs.sigma * sqrt(-log1p(-u1)));
    float s, c;
    sincospif((float)(2.0 * u2), &s, &c);
    y.x += amp * c;
    y.y += amp * s;
  }
  return y;
}

__global__ void k_synth(SynthParams sp, int T, int P, int N, float2* frames,
                        double* truth) {
  const int64_t total = (int64_t)T * P * N;
  const int K = sp.camp.n_targets;
  const double inv_n = 1.0 / (double)N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(e % N);
    const int p = (int)((e / N) % P);
    const int64_t t = e / ((int64_t)N * P);
    RowSynth rs;
    row_setup(sp, P, p, sp.trial0 + (uint64_t)t, rs, sp.err_flag_d);
    if (!sp.wrap)
      for (int k = 0; k < K; ++k)
        if (!(rs.r[k] >= 0.0 && rs.r[k] < (double)N)) atomicOr(sp.err_flag_d, 1);
    frames[e] = synth_sample(rs, K, n, inv_n);
    if (truth && p == 0 && n == 0) {
      // positions re-drawn exactly as row_setup does
      const uint64_t key = substream(sp.camp.seed, sp.trial0 + (uint64_t)t, kSceneTag);
      const int D = sp.camp.dims;
      for (int k = 0; k < K; ++k)
        for (int d = 0; d < 3; ++d) {
          double v = sp.camp.area_lo[d];
          if (d < D) {
            const double u = uniform01(key, (uint64_t)(k * D + d));
            v = __dadd_rn(sp.camp.area_lo[d],
                          __dmul_rn(__dsub_rn(sp.camp.area_hi[d], sp.camp.area_lo[d]), u));
          }
          truth[((int64_t)t * K + k) * 3 + d] = v;
        }
    }
  }
}

// ------------------------------------------------------------ FFT core

// cos / sin of 2 pi e / 16
__device__ constexpr float kC16[16] = {1.0f, 0.92387953251f, 0.70710678118f, 0.38268343236f,
                                       0.0f, -0.38268343236f, -0.70710678118f, -0.92387953251f,
                                       -1.0f, -0.92387953251f, -0.70710678118f, -0.38268343236f,
                                       0.0f, 0.38268343236f, 0.70710678118f, 0.92387953251f};
__device__ constexpr float kS16[16] = {0.0f, 0.38268343236f, 0.70710678118f, 0.92387953251f,
                                       1.0f, 0.92387953251f, 0.70710678118f, 0.38268343236f,
                                       0.0f, -0.38268343236f, -0.70710678118f, -0.92387953251f,
                                       -1.0f, -0.92387953251f, -0.70710678118f, -0.38268343236f};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

constexpr int log2_c(int v) { return v <= 1 ? 0 : 1 + log2_c(v / 2); }

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// x * W16^e (e a compile-time constant after unrolling)
__device__ __forceinline__ float2 w16(float2 x, int e) {
  e &= 15;
  if (e == 0) return x;
  if (e == 4) return make_float2(x.y, -x.x);   // * -i
  if (e == 8) return make_float2(-x.x, -x.y);  // * -1
  if (e == 12) return make_float2(-x.y, x.x);  // * +i
  return cmul(x, make_float2(kC16[e], -kS16[e]));
}

// in-place forward 4-point DFT, natural order
__device__ __forceinline__ void dft4(float2& a, float2& b, float2& c, float2& d) {
  const float2 t0 = cadd(a, c), t1 = csub(a, c);
  const float2 t2 = cadd(b, d), u = csub(b, d);
  const float2 t3 = make_float2(u.y, -u.x);  // (b - d) * -i
  a = cadd(t0, t2);
  c = csub(t0, t2);
  b = cadd(t1, t3);
  d = csub(t1, t3);
}

// Forward R-point DFT in registers, natural order in and out. Written as
// explicit 4x4 / 2x4 factorisations with linear constant indices only: a
// runtime-looking permutation index (bit reversal in a loop) would demote
// v[] to local memory.
template <int R>
__device__ __forceinline__ void dft_reg(float2* v) {
  if constexpr (R == 2) {
    const float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    dft4(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 8) {
    // n = 2 n1 + n2, k = k1 + 4 k2
    float2 y[8];
#pragma unroll
    for (int n2 = 0; n2 < 2; ++n2) {
      float2 a = v[n2], b = v[2 + n2], c = v[4 + n2], d = v[6 + n2];
      dft4(a, b, c, d);
      y[0 * 2 + n2] = a;
      y[1 * 2 + n2] = w16(b, 2 * n2 * 1);
      y[2 * 2 + n2] = w16(c, 2 * n2 * 2);
      y[3 * 2 + n2] = w16(d, 2 * n2 * 3);
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      const float2 a = y[k1 * 2], b = y[k1 * 2 + 1];
      v[k1] = cadd(a, b);
      v[k1 + 4] = csub(a, b);
    }
  } else {
    static_assert(R == 16, "radix 2, 4, 8 or 16");
    // n = 4 n1 + n2, k = k1 + 4 k2
    float2 y[16];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
      float2 a = v[n2], b = v[4 + n2], c = v[8 + n2], d = v[12 + n2];
      dft4(a, b, c, d);
      y[0 * 4 + n2] = a;
      y[1 * 4 + n2] = w16(b, n2 * 1);
      y[2 * 4 + n2] = w16(c, n2 * 2);
      y[3 * 4 + n2] = w16(d, n2 * 3);
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      float2 a = y[k1 * 4 + 0], b = y[k1 * 4 + 1], c = y[k1 * 4 + 2], d = y[k1 * 4 + 3];
      dft4(a, b, c, d);
      v[k1] = a;
      v[k1 + 4] = b;
      v[k1 + 8] = c;
      v[k1 + 12] = d;
    }
  }
}

__device__ __forceinline__ int padi(int i) { return i + (i >> 4); }

struct FftArgs {
  const float2* frames;  // [T][P][N] (or null with synth)
  SynthParams sp;
  int synth;
  int T, P, N, M, os, log2os, log2n, log2m;
  int tb, rows, log2rows, pitch;
  int npass;
  int pass_log2r[8];     // radix (log2) of each Stockham pass
  int out_kind;
  const float2* tw;      // W_M^e = exp(-2 pi i e / M), e < M (global, L1-cached)
  void* out;
};

// One Stockham pass of radix R over every (row, sub-FFT) of the CTA, out of
// place src -> dst (ping-pong buffers: no registers live across barriers).
// ptw: this pass's twiddles W_{Ns R}^{r k} laid out [k][r-1], so lanes with
// consecutive k read with stride (R-1) float2 — bank-conflict free.
template <int R>
__device__ __forceinline__ void stockham_pass(const float2* src, float2* dst, const float2* ptw,
                                              const FftArgs& a, int log2ns, int rows_os) {
  constexpr int LR = log2_c(R);
  const int log2per = a.log2n - LR;
  const int per = 1 << log2per;
  const int Ns = 1 << log2ns;
  const int tasks = rows_os << log2per;
  for (int task = threadIdx.x; task < tasks; task += kFftThreads) {
    const int ro = task >> log2per, q = task & (per - 1);  // ro = row * os + sub
    const int row = ro >> a.log2os, sub = ro & (a.os - 1);
    const int base = row * a.pitch;
    const int off = sub << a.log2n;
    const int k = q & (Ns - 1);
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float2 x = src[base + padi(off + q + r * per)];
      if (r > 0 && Ns > 1) x = cmul(x, ptw[k * (R - 1) + r - 1]);
      v[r] = x;
    }
    dft_reg<R>(v);
    const int o = ((q - k) << LR) + k;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[base + padi(off + o + (r << log2ns))] = v[r];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kFftThreads, 1) k_fft(FftArgs a) {
  extern __shared__ float2 smem_dyn[];
  __shared__ RowSynth rsm[16];
  float2* ptw = smem_dyn;                // per-pass twiddles, N - 1 entries
  float2* buf0 = smem_dyn + a.N;         // rows x pitch, ping
  float2* buf1 = buf0 + a.rows * a.pitch;  // pong
  float2* sm = buf0;
  const int tb = blockIdx.x, p = blockIdx.y;
  const int R = a.rows, M = a.M, N = a.N;
  const double inv_n = 1.0 / (double)N;
  // pass tables: pass with stride Ns and radix Rp holds W_M^{r k M/(Ns Rp)}
  // at [k][r-1] (k < Ns, 1 <= r < Rp); the first pass (Ns = 1) needs none
  {
    int toff = 0, lns = 0;
    for (int ps = 0; ps < a.npass; ++ps) {
      const int lr = a.pass_log2r[ps], rp = 1 << lr, ns = 1 << lns;
      const int cnt = ns * (rp - 1);
      const int step = a.log2m - lns - lr;  // M / (Ns Rp) = 2^step
      for (int e = threadIdx.x; e < cnt; e += kFftThreads) {
        const int k = e / (rp - 1), r = e - k * (rp - 1) + 1;
        ptw[toff + e] = __ldg(a.tw + ((r * k) << step));
      }
      toff += cnt;
      lns += lr;
    }
  }
  for (int g0 = 0; g0 < a.tb; g0 += R) {
    if (a.synth && threadIdx.x < R) {
      const int t = tb * a.tb + g0 + threadIdx.x;
      if (t < a.T) {
        row_setup(a.sp, a.P, p, a.sp.trial0 + (uint64_t)t, rsm[threadIdx.x], a.sp.err_flag_d);
        if (!a.sp.wrap)
          for (int k = 0; k < a.sp.camp.n_targets; ++k) {
            const double r = rsm[threadIdx.x].r[k];
            if (!(r >= 0.0 && r < (double)N)) atomicOr(a.sp.err_flag_d, 1);
          }
      }
    }
    __syncthreads();
    // load: sample n of row r -> sub-FFT j input y[n] W_M^{jn}
    for (int e = threadIdx.x; e < R * N; e += kFftThreads) {
      const int r = e >> a.log2n;
      const int n = e & (N - 1);
      const int t = tb * a.tb + g0 + r;
      float2 v = make_float2(0.f, 0.f);
      if (t < a.T) {
        if (a.synth)
          v = synth_sample(rsm[r], a.sp.camp.n_targets, n, inv_n);
        else
          v = a.frames[((int64_t)t * a.P + p) * N + n];
      }
      float2* row = buf0 + r * a.pitch;
      row[padi(n)] = v;
      for (int j = 1; j < a.os; ++j) row[padi(j * N + n)] = cmul(v, __ldg(a.tw + j * n));
    }
    __syncthreads();
    // N-point Stockham passes, ping-pong between buf0 and buf1
    const int rows_os = R * a.os;
    float2* src = buf0;
    float2* dst = buf1;
    int lns = 0, toff = 0;
    for (int ps = 0; ps < a.npass; ++ps) {
      const int lr = a.pass_log2r[ps];
      const float2* t = ptw + toff;
      if (lr == 4) stockham_pass<16>(src, dst, t, a, lns, rows_os);
      else if (lr == 3) stockham_pass<8>(src, dst, t, a, lns, rows_os);
      else if (lr == 2) stockham_pass<4>(src, dst, t, a, lns, rows_os);
      else stockham_pass<2>(src, dst, t, a, lns, rows_os);
      toff += (1 << lns) * ((1 << lr) - 1);
      lns += lr;
      float2* tmp = src;
      src = dst;
      dst = tmp;
    }
    sm = src;  // result
    // epilogue: output bin k = os * m + j lives in sub-row j at m
    if (a.out_kind == FFT_NATURAL) {
      float2* out = static_cast<float2*>(a.out);
      for (int e = threadIdx.x; e < R * M; e += kFftThreads) {
        const int r = e >> a.log2m, k = e & (M - 1);
        const int t = tb * a.tb + g0 + r;
        const int j = k & (a.os - 1), m = k >> a.log2os;
        if (t < a.T) out[((int64_t)t * a.P + p) * M + k] = sm[r * a.pitch + padi(j * N + m)];
      }
    } else {
      const int64_t base = ((int64_t)tb * a.P + p) * M;
      for (int e = threadIdx.x; e < R * M; e += kFftThreads) {
        const int k = e >> a.log2rows, r = e & (R - 1);
        const int j = k & (a.os - 1), m = k >> a.log2os;
        const float2 z = sm[r * a.pitch + padi(j * N + m)];
        const int64_t o = (base + k) * a.tb + g0 + r;
        if (a.out_kind == FFT_GATHER_COMPLEX) {
          static_cast<float2*>(a.out)[o] = z;
        } else {
          const float pw = z.x * z.x + z.y * z.y;
          static_cast<float*>(a.out)[o] = (a.out_kind == FFT_GATHER_MAG) ? sqrtf(pw) : pw;
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ fixed-size FFT
// The same algorithm with N, os and the rows per pass as compile-time
// constants (the BASELINE sizes): every shared-memory offset folds into an
// immediate, which removes the index arithmetic that dominates the generic
// kernel's instruction count.
__host__ __device__ constexpr int pad_c(int i) { return i + (i >> 4); }

constexpr int kFxThreads = 256;

template <int LN, int LOS, int LROWS>
struct Fx {
  static constexpr int N = 1 << LN, OS = 1 << LOS, M = N * OS, ROWS = 1 << LROWS;
  // padded sub-FFT stride, SUBP = 16/os (mod 16) float2: the os sub-rows
  // holding consecutive output bins k = os*m + j land 32/os banks apart, so
  // the epilogue's reads (consecutive k across lanes) are conflict-free
  static constexpr int SUBP_BASE = N + N / 16;
  static constexpr int SUBP_WANT = OS > 1 ? 16 / OS : 0;
  static constexpr int SUBP = SUBP_BASE + ((SUBP_WANT - SUBP_BASE % 16) + 16) % 16;
  static constexpr int PITCH = OS * SUBP + ((OS * SUBP) % 2 == 0 ? 1 : 0);
  static constexpr int NP = (LN + 3) / 4;
  static constexpr int lr(int ps) { return LN - 4 * ps >= 4 ? 4 : LN - 4 * ps; }
  static constexpr size_t smem_bytes() { return (2ull * ROWS * PITCH + N) * 8; }
  static_assert(LN >= 4, "fixed FFT needs N >= 16");
};

template <int LN, int LOS, int LROWS, int PS>
__device__ __forceinline__ void fixed_pass(const float2* __restrict__ src, float2* __restrict__ dst,
                                           const float2* __restrict__ ptw) {
  using F = Fx<LN, LOS, LROWS>;
  constexpr int LRR = F::lr(PS), R = 1 << LRR, NS = 1 << (4 * PS);
  constexpr int PER = F::N / R;
  constexpr int TASKS = F::ROWS * F::OS * PER;
  constexpr int TW0 = (1 << (4 * PS)) - 1;  // sum of previous radix-16 tables
#pragma unroll
  for (int it = 0; it < (TASKS + kFxThreads - 1) / kFxThreads; ++it) {
    const int task = threadIdx.x + it * kFxThreads;
    if (TASKS % kFxThreads != 0 && task >= TASKS) break;
    const int ro = task / PER, q = task % PER;
    const int row = ro >> LOS, sub = ro & (F::OS - 1);
    const int sbase = row * F::PITCH + sub * F::SUBP;
    const int k = q & (NS - 1);
    float2 v[R];
    if constexpr (PER % 16 == 0) {
      const float2* s = src + sbase + pad_c(q);
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = s[r * (PER + PER / 16)];
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = src[sbase + pad_c(q + r * PER)];
    }
    if constexpr (PS > 0) {
      const float2* t = ptw + TW0 + k * (R - 1);
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], t[r - 1]);
    }
    dft_reg<R>(v);
    const int o = (q - k) * R + k;
    if constexpr (NS % 16 == 0) {
      float2* d = dst + sbase + pad_c(o);
#pragma unroll
      for (int r = 0; r < R; ++r) d[r * (NS + NS / 16)] = v[r];
    } else {
      // first pass: o = q * R is a multiple of 16 and r < 16
      float2* d = dst + sbase + pad_c(o);
#pragma unroll
      for (int r = 0; r < R; ++r) d[r] = v[r];
    }
  }
  __syncthreads();
}

template <int LN, int LOS, int LROWS, int PS>
__device__ __forceinline__ float2* fixed_passes(float2* src, float2* dst, const float2* ptw) {
  using F = Fx<LN, LOS, LROWS>;
  if constexpr (PS < F::NP) {
    fixed_pass<LN, LOS, LROWS, PS>(src, dst, ptw);
    return fixed_passes<LN, LOS, LROWS, PS + 1>(dst, src, ptw);
  } else {
    return src;
  }
}

template <int LN, int LOS, int LROWS>
__global__ void __launch_bounds__(kFxThreads) k_fft_fixed(FftArgs a) {
  using F = Fx<LN, LOS, LROWS>;
  constexpr int N = F::N, M = F::M, R = F::ROWS;
  extern __shared__ float2 smem_dyn[];
  __shared__ RowSynth rsm[16];
  float2* ptw = smem_dyn;
  float2* buf0 = smem_dyn + N;
  float2* buf1 = buf0 + R * F::PITCH;
  const int tb = blockIdx.x, p = blockIdx.y;
  const double inv_n = 1.0 / (double)N;
  {
    int toff = 0;
#pragma unroll
    for (int ps = 1; ps < F::NP; ++ps) {
      const int lr = F::lr(ps), rp = 1 << lr, lns = 4 * ps, ns = 1 << lns;
      toff = (1 << lns) - 1;
      const int cnt = ns * (rp - 1);
      const int step = LN + LOS - lns - lr;
      for (int e = threadIdx.x; e < cnt; e += kFxThreads) {
        const int k = e / (rp - 1), r = e - k * (rp - 1) + 1;
        ptw[toff + e] = __ldg(a.tw + ((r * k) << step));
      }
    }
  }
  // frames of the next row group are fetched into registers while the
  // current group runs its passes (hides the HBM latency behind barriers)
  constexpr int LPT = (R * N + kFxThreads - 1) / kFxThreads;
  float2 pre[LPT];
  auto fetch = [&](int g) {
#pragma unroll
    for (int u = 0; u < LPT; ++u) {
      const int e = threadIdx.x + u * kFxThreads;
      float2 v = make_float2(0.f, 0.f);
      if (e < R * N) {
        const int t = tb * a.tb + g + (e >> LN);
        if (t < a.T) v = __ldg(a.frames + ((int64_t)t * a.P + p) * N + (e & (N - 1)));
      }
      pre[u] = v;
    }
  };
  if (!a.synth) fetch(0);
  for (int g0 = 0; g0 < a.tb; g0 += R) {
    if (a.synth && threadIdx.x < R) {
      const int t = tb * a.tb + g0 + threadIdx.x;
      if (t < a.T) {
        row_setup(a.sp, a.P, p, a.sp.trial0 + (uint64_t)t, rsm[threadIdx.x], a.sp.err_flag_d);
        if (!a.sp.wrap)
          for (int k = 0; k < a.sp.camp.n_targets; ++k) {
            const double r = rsm[threadIdx.x].r[k];
            if (!(r >= 0.0 && r < (double)N)) atomicOr(a.sp.err_flag_d, 1);
          }
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < LPT; ++u) {
      const int e = threadIdx.x + u * kFxThreads;
      if (e >= R * N) break;
      const int r = e >> LN;
      const int n = e & (N - 1);
      float2 v = pre[u];
      if (a.synth) {
        const int t = tb * a.tb + g0 + r;
        v = t < a.T ? synth_sample(rsm[r], a.sp.camp.n_targets, n, inv_n) : make_float2(0.f, 0.f);
      }
      float2* row = buf0 + r * F::PITCH + pad_c(n);
      row[0] = v;
#pragma unroll
      for (int j = 1; j < F::OS; ++j) row[j * F::SUBP] = cmul(v, __ldg(a.tw + j * n));
    }
    if (!a.synth && g0 + R < a.tb) fetch(g0 + R);
    __syncthreads();
    const float2* sm = fixed_passes<LN, LOS, LROWS, 0>(buf0, buf1, ptw);
    if (a.out_kind == FFT_NATURAL) {
      float2* out = static_cast<float2*>(a.out);
      for (int e = threadIdx.x; e < R * M; e += kFxThreads) {
        const int r = e / M, k = e % M;
        const int t = tb * a.tb + g0 + r;
        const int j = k & (F::OS - 1), m = k >> LOS;
        if (t < a.T) out[((int64_t)t * a.P + p) * M + k] = sm[r * F::PITCH + j * F::SUBP + pad_c(m)];
      }
    } else {
      // one thread per range bin k: the R rows' values are contiguous in the
      // gather layout [batch][pair][k][TB] -> vector stores
      const int64_t base = ((int64_t)tb * a.P + p) * M;
#pragma unroll 2
      for (int k = threadIdx.x; k < M; k += kFxThreads) {
        const int j = k & (F::OS - 1), m = k >> LOS;
        const float2* s = sm + j * F::SUBP + pad_c(m);
        float2 z[R];
#pragma unroll
        for (int r = 0; r < R; ++r) z[r] = s[r * F::PITCH];
        const int64_t o = (base + k) * a.tb + g0;
        if (a.out_kind == FFT_GATHER_COMPLEX) {
          float2* dst = static_cast<float2*>(a.out) + o;
          if constexpr (R % 2 == 0) {
#pragma unroll
            for (int r = 0; r < R; r += 2)
              *reinterpret_cast<float4*>(dst + r) = make_float4(z[r].x, z[r].y, z[r + 1].x, z[r + 1].y);
          } else {
            dst[0] = z[0];
          }
        } else {
          float w[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const float pw = z[r].x * z[r].x + z[r].y * z[r].y;
            w[r] = (a.out_kind == FFT_GATHER_MAG) ? sqrtf(pw) : pw;
          }
          float* dst = static_cast<float*>(a.out) + o;
          if constexpr (R % 4 == 0) {
#pragma unroll
            for (int r = 0; r < R; r += 4)
              *reinterpret_cast<float4*>(dst + r) = make_float4(w[r], w[r + 1], w[r + 2], w[r + 3]);
          } else if constexpr (R == 2) {
            *reinterpret_cast<float2*>(dst) = make_float2(w[0], w[1]);
          } else {
            dst[0] = w[0];
          }
        }
      }
    }
    __syncthreads();
  }
}

int ilog2(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}

using FftKernel = void (*)(FftArgs);

// compile-time instantiations: (log2 N, log2 os, log2 rows per pass); rows *
// M = 4096 points per pass keeps a CTA near 70 KB (three CTAs per SM)
FftKernel fixed_kernel(int ln, int los, int lrows, size_t* smem) {
#define GH_FX(a, b, c)                              \
  if (ln == a && los == b && lrows == c) {          \
    *smem = Fx<a, b, c>::smem_bytes();              \
    return k_fft_fixed<a, b, c>;                    \
  }
  GH_FX(6, 2, 4)   // N=64,   M=256  (small test scenes)
  GH_FX(7, 0, 4)   // N=128,  M=128
  GH_FX(8, 2, 2)   // N=256,  M=1024 (c1, c2)
  GH_FX(9, 1, 2)   // N=512,  M=1024 (c4)
  GH_FX(9, 2, 1)   // N=512,  M=2048 (c5)
  GH_FX(10, 2, 0)  // N=1024, M=4096 (c3)
#undef GH_FX
  return nullptr;
}

const float2* twiddles(Ctx* ctx, int M) {
  if (ctx->twiddle_m != M) {
    std::vector<float2> h(static_cast<size_t>(M));
    for (int k = 0; k < M; ++k) {
      const double a = -2.0 * 3.141592653589793238462643383279502884 * k / M;
      h[static_cast<size_t>(k)] = make_float2((float)cos(a), (float)sin(a));
    }
    void* d = ctx->twiddle_buf.get(sizeof(float2) * h.size());
    GH_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(float2) * h.size(), cudaMemcpyHostToDevice,
                            ctx->stream));
    GH_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->twiddle_m = M;
  }
  return static_cast<const float2*>(ctx->twiddle_buf.p);
}

}  // namespace

void launch_fft(Ctx* ctx, const float2* frames_d, const SynthParams* synth, int T, int P,
                int N, int os, int tb, int out_kind, void* out_d) {
  const int M = N * os;
  if ((N & (N - 1)) || (os & (os - 1)) || N < 2)
    fail(GH_EINVAL, "spectra: n_samples and os_range must be powers of two");
  if (M > 16384) fail(GH_EINVAL, "spectra: FFT length above 16384 unsupported");
  if (tb < 1 || tb > 32 || (tb & (tb - 1))) fail(GH_EINVAL, "spectra: bad trial batch");
  FftArgs a{};
  a.frames = frames_d;
  a.synth = synth != nullptr;
  if (synth) a.sp = *synth;
  a.T = T;
  a.P = P;
  a.N = N;
  a.M = M;
  a.os = os;
  a.log2os = ilog2(os);
  a.log2n = ilog2(N);
  a.tb = tb;
  // rows per pass: two padded row buffers + the twiddle table in ~200 KB
  int R = tb < 16 ? tb : 16;
  const int pitch = M + M / 16 + 1;  // padded row, odd in float2 units
  auto bytes = [&](int r) {
    return (2 * static_cast<size_t>(r) * pitch + N) * sizeof(float2);
  };
  while (R > 1 && bytes(R) > 200 * 1024) R >>= 1;
  if (bytes(R) > 220 * 1024) fail(GH_EINVAL, "spectra: FFT too long for one CTA");
  a.rows = R;
  a.log2rows = ilog2(R);
  a.log2m = ilog2(M);
  a.pitch = pitch;
  // radix-16 passes, then one radix-8/4/2 pass for the remainder
  a.npass = 0;
  for (int rem = a.log2n; rem > 0;) {
    const int lr = rem >= 4 ? 4 : rem;
    a.pass_log2r[a.npass++] = lr;
    rem -= lr;
  }
  a.out_kind = out_kind;
  a.tw = twiddles(ctx, M);
  a.out = out_d;
  size_t smem = bytes(R);
  int threads = kFftThreads;
  // fixed-size kernel when this (N, os) has one: rows * M = 4096
  int fr = 1;
  while (fr * 2 <= (tb < 16 ? tb : 16) && fr * 2 * M <= 4096) fr *= 2;
  size_t fsmem = 0;
  FftKernel kern = fixed_kernel(a.log2n, a.log2os, ilog2(fr), &fsmem);
  if (kern) {
    a.rows = fr;
    a.log2rows = ilog2(fr);
    smem = fsmem;
    threads = kFxThreads;
  } else {
    kern = k_fft;
  }
  GH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  const int n_tb = (T + tb - 1) / tb;
  dim3 grid(n_tb, P);
  KTimer kt(ctx, synth ? "synth_fft" : "fft");
  kern<<<grid, threads, smem, ctx->stream>>>(a);
  GH_LAUNCHED(ctx);
}

void launch_synth(Ctx* ctx, const SynthParams& sp, int T, int P, int N, float2* frames_d,
                  double* truth_d) {
  if (sp.camp.n_targets < 1 || sp.camp.n_targets > kMaxTargets)
    fail(GH_EINVAL, "campaign: n_targets must be in [1, 8]");
  if (sp.camp.dims != 2 && sp.camp.dims != 3) fail(GH_EINVAL, "campaign: dims must be 2 or 3");
  const int64_t total = (int64_t)T * P * N;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  KTimer kt(ctx, "synth");
  k_synth<<<blocks, 256, 0, ctx->stream>>>(sp, T, P, N, frames_d, truth_d);
  GH_LAUNCHED(ctx);
}

}  // namespace gh
