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

#include <algorithm>

#include "gh_internal.cuh"
#include "gh_ptx.cuh"

namespace gh {
namespace {

using namespace ptx;

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
    // the counter-based draws are the oracle's bit for bit; the Rayleigh
    // transform runs in fp32 (1 - u1 formed exactly in fp64, >= 2^-53, so
    // the log stays finite): ~1e-7 relative, inside the 2e-5 frame tolerance
    const double u1 = uniform01(rs.noise_key, 2ull * n);
    const double u2 = uniform01(rs.noise_key, 2ull * n + 1);
    const float amp = (float)rs.sigma * sqrtf(-logf((float)(1.0 - u1)));
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

// add_noise (synth.cpp:39-49) on caller frames, complex128 [T][P][N]: the
// synthesis' noise draws (substream (seed, trial, p), draws 2n and 2n + 1;
// rng.hpp complex_gaussian) in fp64, sigma = 10^(-snr / 20) (alpha_ref 1)
__global__ void k_add_noise(double2* frames, int T, int P, int N, uint64_t seed, uint64_t trial0,
                            double sigma) {
  const int64_t total = (int64_t)T * P * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(e % N);
    const int p = (int)((e / N) % P);
    const int64_t t = e / ((int64_t)N * P);
    const uint64_t key = substream(seed, trial0 + (uint64_t)t, (uint64_t)p);
    const double u1 = uniform01(key, 2ull * n), u2 = uniform01(key, 2ull * n + 1);
    const double amp = sigma * sqrt(-log1p(-u1));
    double s, c;
    sincospi(2.0 * u2, &s, &c);
    frames[e].x += amp * c;
    frames[e].y += amp * s;
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
// The BASELINE sizes run a compile-time specialisation that works on two
// rows (trials) at once with sm_100's packed fp32 instructions: a point of
// a row pair is one float4 {re_a, re_b, im_a, im_b}, so every complex add is
// two FADD2 and every twiddle product four FMUL2/FFMA2 (the twiddle is a
// scalar-broadcast operand) for two trials — half the FP instructions and
// half the shared-memory instructions of a per-row FFT. Each thread owns
// exactly 16 points of every pass (one radix-16 task, or 16/R radix-R
// tasks), so the passes run in place: load, DFT in registers, barrier,
// store, barrier. All shared-memory offsets fold into immediates.
__host__ __device__ constexpr int pad_c(int i) { return i + (i >> 4); }

struct Cx2 {  // one complex point of two rows: re = (a, b), im = (a, b)
  float2 re, im;
};
__device__ __forceinline__ Cx2 cx_add(Cx2 a, Cx2 b) {
  return {__fadd2_rn(a.re, b.re), __fadd2_rn(a.im, b.im)};
}
__device__ __forceinline__ Cx2 cx_sub(Cx2 a, Cx2 b) {
  return {__fadd2_rn(a.re, make_float2(-b.re.x, -b.re.y)),
          __fadd2_rn(a.im, make_float2(-b.im.x, -b.im.y))};
}
// x * (c + i s), c and s broadcast to both rows
__device__ __forceinline__ Cx2 cx_mul(Cx2 x, float c, float s) {
  return {__ffma2_rn(x.im, make_float2(-s, -s), __fmul2_rn(x.re, make_float2(c, c))),
          __ffma2_rn(x.im, make_float2(c, c), __fmul2_rn(x.re, make_float2(s, s)))};
}
__device__ __forceinline__ Cx2 cx_mul_mi(Cx2 x) {  // x * -i
  return {x.im, make_float2(-x.re.x, -x.re.y)};
}
__device__ __forceinline__ Cx2 cx_w16(Cx2 x, int e) {  // x * W16^e, e constant
  e &= 15;
  if (e == 0) return x;
  if (e == 4) return cx_mul_mi(x);
  if (e == 8) return {make_float2(-x.re.x, -x.re.y), make_float2(-x.im.x, -x.im.y)};
  if (e == 12) return {make_float2(-x.im.x, -x.im.y), x.re};
  return cx_mul(x, kC16[e], -kS16[e]);
}
__device__ __forceinline__ void cx_dft4(Cx2& a, Cx2& b, Cx2& c, Cx2& d) {
  const Cx2 t0 = cx_add(a, c), t1 = cx_sub(a, c);
  const Cx2 t2 = cx_add(b, d), t3 = cx_mul_mi(cx_sub(b, d));
  a = cx_add(t0, t2);
  c = cx_sub(t0, t2);
  b = cx_add(t1, t3);
  d = cx_sub(t1, t3);
}
// forward R-point DFT, natural order in and out (same factorisations as
// dft_reg, constant indices only)
template <int R>
__device__ __forceinline__ void cx_dft(Cx2* v) {
  if constexpr (R == 2) {
    const Cx2 a = v[0], b = v[1];
    v[0] = cx_add(a, b);
    v[1] = cx_sub(a, b);
  } else if constexpr (R == 4) {
    cx_dft4(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 8) {
    Cx2 y[8];
#pragma unroll
    for (int n2 = 0; n2 < 2; ++n2) {
      Cx2 a = v[n2], b = v[2 + n2], c = v[4 + n2], d = v[6 + n2];
      cx_dft4(a, b, c, d);
      y[0 * 2 + n2] = a;
      y[1 * 2 + n2] = cx_w16(b, 2 * n2 * 1);
      y[2 * 2 + n2] = cx_w16(c, 2 * n2 * 2);
      y[3 * 2 + n2] = cx_w16(d, 2 * n2 * 3);
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      const Cx2 a = y[k1 * 2], b = y[k1 * 2 + 1];
      v[k1] = cx_add(a, b);
      v[k1 + 4] = cx_sub(a, b);
    }
  } else {
    static_assert(R == 16, "radix 2, 4, 8 or 16");
    Cx2 y[16];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
      Cx2 a = v[n2], b = v[4 + n2], c = v[8 + n2], d = v[12 + n2];
      cx_dft4(a, b, c, d);
      y[0 * 4 + n2] = a;
      y[1 * 4 + n2] = cx_w16(b, n2 * 1);
      y[2 * 4 + n2] = cx_w16(c, n2 * 2);
      y[3 * 4 + n2] = cx_w16(d, n2 * 3);
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      Cx2 a = y[k1 * 4 + 0], b = y[k1 * 4 + 1], c = y[k1 * 4 + 2], d = y[k1 * 4 + 3];
      cx_dft4(a, b, c, d);
      v[k1] = a;
      v[k1 + 4] = b;
      v[k1 + 8] = c;
      v[k1 + 12] = d;
    }
  }
}
__device__ __forceinline__ Cx2 cx_ld(const float4* p) {
  const float4 q = *p;
  return {make_float2(q.x, q.y), make_float2(q.z, q.w)};
}
// two 8-byte stores: the DFT leaves re and im in unrelated register pairs,
// and one 16-byte store would cost two register moves per point
// (inline PTX: the compiler would merge the pair back into one STS.128)
__device__ __forceinline__ void cx_st(float4* p, Cx2 v) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.re.x), "f"(v.re.y) : "memory");
  asm volatile("st.shared.v2.f32 [%0+8], {%1, %2};" ::"r"(a), "f"(v.im.x), "f"(v.im.y) : "memory");
}

// LN = log2 N, LOS = log2 os, LP = log2 row pairs per group
template <int LN, int LOS, int LP>
struct Fx {
  static constexpr int N = 1 << LN, OS = 1 << LOS, M = N * OS, PAIRS = 1 << LP, ROWS = 2 * PAIRS;
  static constexpr int THREADS = PAIRS * M / 16;  // 16 points of every pass per thread
  // padded sub-FFT stride in float4, SUBP = 8/os (mod 8): the os sub-rows
  // holding consecutive output bins k = os*m + j land in distinct 16-byte
  // bank groups, so the epilogue's reads (consecutive k across lanes) are
  // conflict-free
  static constexpr int SUBP_BASE = N + N / 16;
  static constexpr int SUBP_WANT = OS > 1 ? 8 / OS : 0;
  static constexpr int SUBP = SUBP_BASE + ((SUBP_WANT - SUBP_BASE % 8) + 8) % 8;
  static constexpr int PITCH = OS * SUBP;  // float4 per row pair
  static constexpr int NP = (LN + 3) / 4;
  static constexpr int lr(int ps) { return LN - 4 * ps >= 4 ? 4 : LN - 4 * ps; }
  static constexpr int TWN = N;             // pass twiddles (< N entries)
  static constexpr int TWL = (OS - 1) * N;   // load twiddles W_M^{jn}, 1 <= j < os
  static constexpr size_t smem_bytes() { return (size_t)PAIRS * PITCH * 16 + (TWN + TWL) * 8; }
  static_assert(LN >= 4 && OS <= 8, "fixed FFT needs N >= 16, os <= 8");
  static_assert(THREADS >= 32 && THREADS <= 1024, "fixed FFT block size");
};

template <int LN, int LOS, int LP, int PS>
__device__ __forceinline__ void fixed_pass(float4* __restrict__ buf, const float2* __restrict__ ptw) {
  using F = Fx<LN, LOS, LP>;
  constexpr int LRR = F::lr(PS), R = 1 << LRR, NS = 1 << (4 * PS);
  constexpr int PER = F::N / R;
  constexpr int TPT = 16 / R;                // tasks per thread
  constexpr int TW0 = (1 << (4 * PS)) - 1;   // sum of previous radix-16 tables
  Cx2 v[TPT][R];
  int sb[TPT], oo[TPT];
#pragma unroll
  for (int it = 0; it < TPT; ++it) {
    const int task = threadIdx.x + it * F::THREADS;
    const int ro = task / PER, q = task % PER;  // ro = pair * os + sub
    const int sbase = (ro >> LOS) * F::PITCH + (ro & (F::OS - 1)) * F::SUBP;
    const int k = q & (NS - 1);
#pragma unroll
    for (int r = 0; r < R; ++r) v[it][r] = cx_ld(buf + sbase + pad_c(q + r * PER));
    if constexpr (PS > 0) {
      const float2* t = ptw + TW0 + k * (R - 1);
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const float2 w = t[r - 1];
        v[it][r] = cx_mul(v[it][r], w.x, w.y);
      }
    }
    cx_dft<R>(v[it]);
    sb[it] = sbase;
    oo[it] = (q - k) * R + k;
  }
  __syncthreads();  // every point of the pass read: overwrite in place
#pragma unroll
  for (int it = 0; it < TPT; ++it) {
#pragma unroll
    for (int r = 0; r < R; ++r) cx_st(buf + sb[it] + pad_c(oo[it] + r * NS), v[it][r]);
  }
  __syncthreads();
}

template <int LN, int LOS, int LP, int PS>
__device__ __forceinline__ void fixed_passes(float4* buf, const float2* ptw) {
  if constexpr (PS < Fx<LN, LOS, LP>::NP) {
    fixed_pass<LN, LOS, LP, PS>(buf, ptw);
    fixed_passes<LN, LOS, LP, PS + 1>(buf, ptw);
  }
}

// epilogue kinds of the fixed kernel (compile time)
enum FxOut { FX_NATURAL = 0, FX_REAL = 1, FX_COMPLEX = 2 };

// c3 (N = 1024, os = 4, one row pair): capped at 128 registers (8 bytes of spills)
// so two CTAs share an SM (102 KB of shared memory each); uncapped it takes 156
// registers and runs one CTA of 8 warps per SM
template <int LN, int LOS, int LP>
constexpr int fixed_min_ctas() { return LN == 10 && LOS == 2 && LP == 0 ? 2 : 1; }

template <int LN, int LOS, int LP, bool SYNTH, int KIND>
__global__ void __launch_bounds__(Fx<LN, LOS, LP>::THREADS, fixed_min_ctas<LN, LOS, LP>())
    k_fft_fixed(FftArgs a) {
  using F = Fx<LN, LOS, LP>;
  constexpr int N = F::N, M = F::M, PAIRS = F::PAIRS, ROWS = F::ROWS, NT = F::THREADS;
  extern __shared__ float4 smem4[];
  __shared__ RowSynth rsm[SYNTH ? ROWS : 1];
  float4* buf = smem4;
  float2* ptw = reinterpret_cast<float2*>(smem4 + PAIRS * F::PITCH);
  float2* ltw = ptw + F::TWN;  // load twiddles W_M^{jn} at [(j-1) N + n]
  const double inv_n = 1.0 / (double)N;
  // pass twiddles: pass ps (stride NS, radix R) holds W_M^{r k M/(NS R)} at
  // [k][r-1]; the first pass needs none
#pragma unroll
  for (int ps = 1; ps < F::NP; ++ps) {
    const int lr = F::lr(ps), rp = 1 << lr, lns = 4 * ps, ns = 1 << lns;
    const int toff = (1 << lns) - 1;
    const int cnt = ns * (rp - 1);
    const int step = LN + LOS - lns - lr;
    for (int e = threadIdx.x; e < cnt; e += NT) {
      const int k = e / (rp - 1), r = e - k * (rp - 1) + 1;
      ptw[toff + e] = __ldg(a.tw + ((r * k) << step));
    }
  }
  for (int e = threadIdx.x; e < (F::OS - 1) * N; e += NT) {
    const int j = e / N + 1, n = e % N;
    ltw[e] = __ldg(a.tw + j * n);
  }
  // Persistent CTAs walk the (trial batch, pair) items; the frames of the
  // next row group — of this item, or the first group of the CTA's next
  // item — are fetched into registers while the current group runs its
  // passes, so no group waits on HBM latency (not even an item's first).
  const int n_tb = (a.T + a.tb - 1) / a.tb;
  const int n_items = n_tb * a.P;
  constexpr int LPT = (PAIRS * N + NT - 1) / NT;
  float2 pre[SYNTH ? 1 : LPT][2];
  auto fetch = [&](int item, int g) {
    const int ftb = item % n_tb, fp = item / n_tb;
    const float2* fr = a.frames + ((int64_t)ftb * a.tb * a.P + fp) * N;  // row r: + r P N
    const int left = a.T - ftb * a.tb;
#pragma unroll
    for (int u = 0; u < LPT; ++u) {
      const int e = threadIdx.x + u * NT;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float2 v = make_float2(0.f, 0.f);
        const int r = g + 2 * (e >> LN) + h;
        if ((PAIRS * N % NT == 0 || e < PAIRS * N) && r < left)
          v = __ldg(fr + (int64_t)r * a.P * N + (e & (N - 1)));
        pre[u][h] = v;
      }
    }
  };
  if constexpr (!SYNTH)
    if ((int)blockIdx.x < n_items) fetch(blockIdx.x, 0);
  __syncthreads();  // twiddle tables
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
  const int tb = item % n_tb, p = item / n_tb;
  const int rows_left = a.T - tb * a.tb;  // rows of this batch that exist
  for (int g0 = 0; g0 < a.tb; g0 += ROWS) {
    if constexpr (SYNTH) {
      if (threadIdx.x < ROWS) {
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
    }
    // load: sample n of the pair's rows -> sub-FFT j input y[n] W_M^{jn}
#pragma unroll
    for (int u = 0; u < LPT; ++u) {
      const int e = threadIdx.x + u * NT;
      if (PAIRS * N % NT != 0 && e >= PAIRS * N) break;
      const int pp = e >> LN;
      const int n = e & (N - 1);
      float2 ya, yb;
      if constexpr (SYNTH) {
        const int r = g0 + 2 * pp;
        const float2 z = make_float2(0.f, 0.f);
        ya = r < rows_left ? synth_sample(rsm[2 * pp], a.sp.camp.n_targets, n, inv_n) : z;
        yb = r + 1 < rows_left ? synth_sample(rsm[2 * pp + 1], a.sp.camp.n_targets, n, inv_n) : z;
      } else {
        ya = pre[u][0];
        yb = pre[u][1];
      }
      const Cx2 y{make_float2(ya.x, yb.x), make_float2(ya.y, yb.y)};
      float4* row = buf + pp * F::PITCH + pad_c(n);
      cx_st(row, y);
#pragma unroll
      for (int j = 1; j < F::OS; ++j) {
        const float2 w = ltw[(j - 1) * N + n];
        cx_st(row + j * F::SUBP, cx_mul(y, w.x, w.y));
      }
    }
    if constexpr (!SYNTH) {
      if (g0 + ROWS < a.tb) fetch(item, g0 + ROWS);
      else if (item + (int)gridDim.x < n_items) fetch(item + gridDim.x, 0);
    }
    __syncthreads();
    fixed_passes<LN, LOS, LP, 0>(buf, ptw);
    // epilogue: output bin k = os * m + j lives in sub-row j at m
    if constexpr (KIND == FX_NATURAL) {
      float2* out = static_cast<float2*>(a.out);
      for (int e = threadIdx.x; e < PAIRS * M; e += NT) {
        const int pp = e / M, k = e % M;
        const int t = tb * a.tb + g0 + 2 * pp;
        const int j = k & (F::OS - 1), m = k >> LOS;
        const Cx2 z = cx_ld(buf + pp * F::PITCH + j * F::SUBP + pad_c(m));
        if (t < a.T) out[((int64_t)t * a.P + p) * M + k] = make_float2(z.re.x, z.im.x);
        if (t + 1 < a.T) out[((int64_t)(t + 1) * a.P + p) * M + k] = make_float2(z.re.y, z.im.y);
      }
    } else {
      // one thread per range bin k: the group's rows are contiguous in the
      // gather layout [batch][pair][k][TB] -> vector stores
      const int64_t o0 = ((int64_t)tb * a.P + p) * M * a.tb + g0;
      const bool mag = a.out_kind == FFT_GATHER_MAG;
#pragma unroll 2
      for (int k = threadIdx.x; k < M; k += NT) {
        const int j = k & (F::OS - 1), m = k >> LOS;
        const float4* s = buf + j * F::SUBP + pad_c(m);
        const int64_t o = o0 + (int64_t)k * a.tb;
        if constexpr (KIND == FX_COMPLEX) {
          float4* dst = reinterpret_cast<float4*>(static_cast<float2*>(a.out) + o);
#pragma unroll
          for (int pp = 0; pp < PAIRS; ++pp) {
            const Cx2 z = cx_ld(s + pp * F::PITCH);
            dst[pp] = make_float4(z.re.x, z.im.x, z.re.y, z.im.y);
          }
        } else {
          float2 w[PAIRS];
#pragma unroll
          for (int pp = 0; pp < PAIRS; ++pp) {
            const Cx2 z = cx_ld(s + pp * F::PITCH);
            w[pp] = __ffma2_rn(z.re, z.re, __fmul2_rn(z.im, z.im));
            if (mag) w[pp] = make_float2(sqrtf(w[pp].x), sqrtf(w[pp].y));
          }
          float* dst = static_cast<float*>(a.out) + o;
          if constexpr (PAIRS % 2 == 0) {
#pragma unroll
            for (int pp = 0; pp < PAIRS; pp += 2)
              *reinterpret_cast<float4*>(dst + 2 * pp) =
                  make_float4(w[pp].x, w[pp].y, w[pp + 1].x, w[pp + 1].y);
          } else {
            *reinterpret_cast<float2*>(dst) = w[0];
          }
        }
      }
    }
    __syncthreads();
  }
  }  // items
}

// ------------------------------------------- N = 256 warp-resident FFT
// The c1/c2 size (N = 256, os = 4, M = 1024) as two register radix-16
// stages with ONE warp-private shared-memory exchange. With n = 16 a + t
// (a, t < 16) and k = 64 k3 + k2:
//   stage 1  Y_t[4 k1 + j] = sum_a (y[16a+t] W_64^{a j}) W_16^{a k1}
//   stage 2  X[64 k3 + k2] = sum_t (Y_t[k2] W_M^{t k2}) W_16^{t k3}
// One row per lane with the complex value packed (re, im) in one fp32x2
// register pair: a complex add is one FADD2 and a twiddle product one
// FMUL2 + one FFMA2 on the swapped pair (sm_100 operand swizzle), so a lane
// holds 16 points in 32 registers and an SM keeps 32 warps resident.
// A CTA (8 warps) walks 4-trial groups of one (batch, pair); warp w owns
// sub-FFT index j = w % 4 of rows 2 (w / 4) + h (h = lane / 16). Lane (t, h)
// runs stage 1 on its 16 stride-16 samples; the exchange hands lane (k1, h)
// the 16 Y_t[4 k1 + j]; stage 2 yields 16 output bins, whose power goes to
// a CTA buffer [k][4 trials] (16-byte chunks XOR-swizzled so the scattered
// 4-byte writes are 2-way at worst); after one barrier every bin leaves as
// one 16-byte store into the gather layout [batch][pair][k][TB]. The
// group's four 2 KB rows arrive by TMA bulk copies into a 2-deep ring (one
// mbarrier per stage): the last warp to read a stage (a shared-memory
// counter) issues the copies of the CTA's group 2 ahead into it, so no warp
// waits as a producer.
// Shared-memory traffic per row: 2 KB input read + one 2 KB exchange each
// way (the Stockham kernel above moves ~28 KB per row).
constexpr int kR16Warps = 8;
constexpr int kR16Xp = 16 * 17;  // float2 per exchange row: [k1][t], pitch 17
constexpr int kR16St = 2;        // input ring stages
constexpr size_t kR16Smem =
    (kR16St * 4 * 256 + kR16Warps * 2 * kR16Xp + 1024 * 2) * sizeof(float2);
__constant__ float2 c_w64[64] = {
    {1.0000000000f, -0.0000000000f}, {0.9951847267f, -0.0980171403f}, {0.9807852804f, -0.1950903220f}, {0.9569403357f, -0.2902846773f},
    {0.9238795325f, -0.3826834324f}, {0.8819212643f, -0.4713967368f}, {0.8314696123f, -0.5555702330f}, {0.7730104534f, -0.6343932842f},
    {0.7071067812f, -0.7071067812f}, {0.6343932842f, -0.7730104534f}, {0.5555702330f, -0.8314696123f}, {0.4713967368f, -0.8819212643f},
    {0.3826834324f, -0.9238795325f}, {0.2902846773f, -0.9569403357f}, {0.1950903220f, -0.9807852804f}, {0.0980171403f, -0.9951847267f},
    {0.0000000000f, -1.0000000000f}, {-0.0980171403f, -0.9951847267f}, {-0.1950903220f, -0.9807852804f}, {-0.2902846773f, -0.9569403357f},
    {-0.3826834324f, -0.9238795325f}, {-0.4713967368f, -0.8819212643f}, {-0.5555702330f, -0.8314696123f}, {-0.6343932842f, -0.7730104534f},
    {-0.7071067812f, -0.7071067812f}, {-0.7730104534f, -0.6343932842f}, {-0.8314696123f, -0.5555702330f}, {-0.8819212643f, -0.4713967368f},
    {-0.9238795325f, -0.3826834324f}, {-0.9569403357f, -0.2902846773f}, {-0.9807852804f, -0.1950903220f}, {-0.9951847267f, -0.0980171403f},
    {-1.0000000000f, -0.0000000000f}, {-0.9951847267f, 0.0980171403f}, {-0.9807852804f, 0.1950903220f}, {-0.9569403357f, 0.2902846773f},
    {-0.9238795325f, 0.3826834324f}, {-0.8819212643f, 0.4713967368f}, {-0.8314696123f, 0.5555702330f}, {-0.7730104534f, 0.6343932842f},
    {-0.7071067812f, 0.7071067812f}, {-0.6343932842f, 0.7730104534f}, {-0.5555702330f, 0.8314696123f}, {-0.4713967368f, 0.8819212643f},
    {-0.3826834324f, 0.9238795325f}, {-0.2902846773f, 0.9569403357f}, {-0.1950903220f, 0.9807852804f}, {-0.0980171403f, 0.9951847267f},
    {-0.0000000000f, 1.0000000000f}, {0.0980171403f, 0.9951847267f}, {0.1950903220f, 0.9807852804f}, {0.2902846773f, 0.9569403357f},
    {0.3826834324f, 0.9238795325f}, {0.4713967368f, 0.8819212643f}, {0.5555702330f, 0.8314696123f}, {0.6343932842f, 0.7730104534f},
    {0.7071067812f, 0.7071067812f}, {0.7730104534f, 0.6343932842f}, {0.8314696123f, 0.5555702330f}, {0.8819212643f, 0.4713967368f},
    {0.9238795325f, 0.3826834324f}, {0.9569403357f, 0.2902846773f}, {0.9807852804f, 0.1950903220f}, {0.9951847267f, 0.0980171403f}};  // W_64^e

__device__ __forceinline__ float2 c1_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 c1_sub(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 c1_mul(float2 x, float2 w) {  // x * w
  return __ffma2_rn(make_float2(x.y, x.x), make_float2(-w.y, w.y),
                    __fmul2_rn(x, make_float2(w.x, w.x)));
}
__device__ __forceinline__ float2 c1_mi(float2 x) { return make_float2(x.y, -x.x); }  // x * -i
__device__ __forceinline__ float2 c1_w16(float2 x, int e) {  // x * W16^e, e constant
  e &= 15;
  if (e == 0) return x;
  if (e == 4) return c1_mi(x);
  if (e == 8) return make_float2(-x.x, -x.y);
  if (e == 12) return make_float2(-x.y, x.x);
  return c1_mul(x, make_float2(kC16[e], -kS16[e]));
}
__device__ __forceinline__ void c1_dft4(float2& a, float2& b, float2& c, float2& d) {
  const float2 t0 = c1_add(a, c), t1 = c1_sub(a, c);
  const float2 t2 = c1_add(b, d), t3 = c1_mi(c1_sub(b, d));
  a = c1_add(t0, t2);
  c = c1_sub(t0, t2);
  b = c1_add(t1, t3);
  d = c1_sub(t1, t3);
}
// forward 16-point DFT, natural order in and out (4 x 4)
__device__ __forceinline__ void c1_dft16(float2* v) {
  float2 y[16];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    float2 a = v[n2], b = v[4 + n2], c = v[8 + n2], d = v[12 + n2];
    c1_dft4(a, b, c, d);
    y[0 * 4 + n2] = a;
    y[1 * 4 + n2] = c1_w16(b, n2 * 1);
    y[2 * 4 + n2] = c1_w16(c, n2 * 2);
    y[3 * 4 + n2] = c1_w16(d, n2 * 3);
  }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    float2 a = y[k1 * 4 + 0], b = y[k1 * 4 + 1], c = y[k1 * 4 + 2], d = y[k1 * 4 + 3];
    c1_dft4(a, b, c, d);
    v[k1] = a;
    v[k1 + 4] = b;
    v[k1 + 8] = c;
    v[k1 + 12] = d;
  }
}

template <bool MAG>
__global__ void __launch_bounds__(kR16Warps * 32, 3) k_fft256(FftArgs a) {
  constexpr int N = 256, M = 1024, K2 = 64;
  extern __shared__ __align__(16) float2 r16[];
  float2* in = r16;                     // [stages][4 rows][256]
  float2* xs = r16 + kR16St * 4 * 256;  // per warp: [h][k1][17]
  float* ob = reinterpret_cast<float*>(xs + kR16Warps * 2 * kR16Xp);  // [k (swizzled)][4]
  __shared__ __align__(8) uint64_t full[kR16St];
  __shared__ int readers[kR16St];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane & 15, h = lane >> 4, j = warp & 3, row = 2 * (warp >> 2) + h;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kR16St; ++s) {
      mbar_init(&full[s], 1);
      readers[s] = 0;
    }
    mbar_fence_init();
  }
  __syncthreads();
  float2* xw = xs + (warp * 2 + h) * kR16Xp;
  // stage-2 twiddles W_M^{t (4 k1 + j)}: per-lane recurrences (step W_M^{4t})
  // re-seeded exactly at k1 = 0 and 8
  const float2 seed0 = __ldg(a.tw + t * j), seed8 = __ldg(a.tw + t * (32 + j));
  const float2 step = __ldg(a.tw + 4 * t);
  const int groups = a.tb >> 2;  // 4-trial groups per batch
  const int n_tb = (a.T + a.tb - 1) / a.tb;
  const int n_items = n_tb * a.P * groups;
  // group g of (batch, pair): rows tb*TB + 4 g + r; rows past T repeat the
  // last trial (finite values; the gather ignores trials >= T)
  auto issue = [&](int item, int s) {
    const int g = item % groups, p = (item / groups) % a.P, tb = item / (groups * a.P);
    mbar_expect_tx(&full[s], 4u * N * sizeof(float2));
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int tr = min(tb * a.tb + 4 * g + r, a.T - 1);
      bulk_g2s(in + (s * 4 + r) * N, a.frames + ((int64_t)tr * a.P + p) * N,
               N * sizeof(float2), &full[s]);
    }
    mbar_arrive(&full[s]);
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < kR16St; ++s)
      if ((int)blockIdx.x + s * (int)gridDim.x < n_items) issue(blockIdx.x + s * gridDim.x, s);
  int it = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
    const int s = it % kR16St;
    const int g = item % groups, p = (item / groups) % a.P, tb = item / (groups * a.P);
    mbar_wait(&full[s], (it / kR16St) & 1);
    const float2* src = in + (s * 4 + row) * N + t;
    float2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = src[16 * q];
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&readers[s], 1) == kR16Warps - 1) {  // last reader refills
        readers[s] = 0;
        const int nx = item + kR16St * (int)gridDim.x;
        if (nx < n_items) issue(nx, s);
      }
    }
    if (j != 0) {
#pragma unroll
      for (int q = 1; q < 16; ++q) v[q] = c1_mul(v[q], c_w64[(q * j) & 63]);
    }
    c1_dft16(v);
    float2 w = seed0;
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) {
      if (k1 == 8) w = seed8;
      xw[k1 * 17 + t] = c1_mul(v[k1], w);
      if (k1 != 7 && k1 != 15) w = c1_mul(w, step);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = xw[t * 17 + q];  // lane t = k1
    __syncwarp();  // the next group overwrites the exchange rows
    c1_dft16(v);
    // v[k3] = X[64 k3 + 4 t + j] of row 2 (warp / 4) + h of the group
#pragma unroll
    for (int k3 = 0; k3 < 16; ++k3) {
      const float2 sq = __fmul2_rn(v[k3], v[k3]);
      const float pw = sq.x + sq.y;
      const int k = 64 * k3 + 4 * t + j;
      ob[4 * (k ^ ((k >> 3) & 7)) + row] = MAG ? sqrtf(pw) : pw;
    }
    __syncthreads();
    float* dst = static_cast<float*>(a.out) + ((int64_t)tb * a.P + p) * M * a.tb + g * 4;
#pragma unroll
    for (int i = 0; i < M / (kR16Warps * 32); ++i) {
      const int k = threadIdx.x + i * kR16Warps * 32;
      *reinterpret_cast<float4*>(dst + (int64_t)k * a.tb) =
          *reinterpret_cast<const float4*>(ob + 4 * (k ^ ((k >> 3) & 7)));
    }
    __syncthreads();  // the next group overwrites ob
  }
}

int ilog2(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}

using FftKernel = void (*)(FftArgs);

template <int LN, int LOS, int LP>
FftKernel fixed_variant(bool synth, int out_kind, size_t* smem, int* threads) {
  *smem = Fx<LN, LOS, LP>::smem_bytes();
  *threads = Fx<LN, LOS, LP>::THREADS;
  const int kind = out_kind == FFT_NATURAL ? FX_NATURAL
                   : out_kind == FFT_GATHER_COMPLEX ? FX_COMPLEX : FX_REAL;
  if (synth) {
    if (kind == FX_NATURAL) return k_fft_fixed<LN, LOS, LP, true, FX_NATURAL>;
    if (kind == FX_COMPLEX) return k_fft_fixed<LN, LOS, LP, true, FX_COMPLEX>;
    return k_fft_fixed<LN, LOS, LP, true, FX_REAL>;
  }
  if (kind == FX_NATURAL) return k_fft_fixed<LN, LOS, LP, false, FX_NATURAL>;
  if (kind == FX_COMPLEX) return k_fft_fixed<LN, LOS, LP, false, FX_COMPLEX>;
  return k_fft_fixed<LN, LOS, LP, false, FX_REAL>;
}

// compile-time instantiations: (log2 N, log2 os, log2 row pairs per group);
// pairs * M = 4096 points (256 threads) where the trial batch allows
FftKernel fixed_kernel(int ln, int los, int lp, bool synth, int out_kind, size_t* smem,
                       int* threads) {
#define GH_FX(a, b, c) \
  if (ln == a && los == b && lp == c) return fixed_variant<a, b, c>(synth, out_kind, smem, threads);
  GH_FX(6, 2, 2)   // N=64,   M=256  (small test scenes, 8-trial batches)
  GH_FX(6, 2, 3)   // N=64,   M=256  (16-trial batches)
  GH_FX(7, 0, 3)   // N=128,  M=128
  GH_FX(8, 2, 2)   // N=256,  M=1024 (c1, c2)
  GH_FX(9, 1, 2)   // N=512,  M=1024 (c4)
  GH_FX(9, 2, 1)   // N=512,  M=2048 (c5)
  GH_FX(10, 2, 0)  // N=1024, M=4096 (c3)
#undef GH_FX
  return nullptr;
}

const float2* twiddles(Ctx* ctx, int M) {
  if (ctx->twiddle_m != M) {
    // [0, M): W_M^k; [M, 2M): W_M^{t k2} at [k2][t], t < 16 (k_fft256)
    std::vector<float2> h(2 * static_cast<size_t>(M));
    for (int k = 0; k < 2 * M; ++k) {
      const int e = k < M ? k : ((k - M) & 15) * ((k - M) >> 4) % M;
      const double a = -2.0 * 3.141592653589793238462643383279502884 * e / M;
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
  // fixed-size row-pair kernel when this (N, os) has one: pairs * M <= 4096,
  // at most 8 pairs, and the trial batch a whole number of row groups
  int lp = -1;
  if (tb >= 2) {
    lp = ilog2(tb) - 1;
    while (lp > 0 && ((M << lp) > 4096 || lp > 3)) --lp;
  }
  if (!synth && N == 256 && os == 4 && tb % 4 == 0 &&
      (out_kind == FFT_GATHER_POWER || out_kind == FFT_GATHER_MAG)) {
    FftKernel k = out_kind == FFT_GATHER_MAG ? k_fft256<true> : k_fft256<false>;
    GH_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kR16Smem)));
    int occ = 0;
    GH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kR16Warps * 32, kR16Smem));
    const int64_t items = (int64_t)((T + tb - 1) / tb) * P * (tb / 4);
    const int64_t blocks =
        std::min<int64_t>(items, (int64_t)std::max(occ, 1) * ctx->num_sms);
    KTimer kt(ctx, "fft");
    k<<<static_cast<unsigned>(blocks), kR16Warps * 32, kR16Smem, ctx->stream>>>(a);
    GH_LAUNCHED(ctx);
    return;
  }
  size_t fsmem = 0;
  int fthreads = 0;
  FftKernel kern = lp >= 0 ? fixed_kernel(a.log2n, a.log2os, lp, synth != nullptr, out_kind,
                                          &fsmem, &fthreads)
                           : nullptr;
  if (kern) {
    smem = fsmem;
    threads = fthreads;
  } else {
    kern = k_fft;
  }
  GH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  const int n_tb = (T + tb - 1) / tb;
  dim3 grid(n_tb, P);
  if (kern != k_fft) {
    // fixed kernels are persistent over the (batch, pair) items
    int occ = 0;
    GH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
    const int64_t items = (int64_t)n_tb * P;
    grid = dim3(static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)std::max(occ, 1) * ctx->num_sms))));
  }
  KTimer kt(ctx, synth ? "synth_fft" : "fft");
  kern<<<grid, threads, smem, ctx->stream>>>(a);
  GH_LAUNCHED(ctx);
}

namespace {

// Multi-chirp frames (the reference's slow-time axis, Mc > 1): power summed
// over a trial's chirps, sum_mc |Z_q(mc, k)|^2, written in the gather layout
// [batch][pair][M][TB]. A CTA owns (batch, pair, 64 range bins): it reads the
// natural spectra [T][P][Mc][M] with consecutive threads on consecutive bins
// (coalesced), accumulates in shared memory and stores each bin's TB-run
// contiguously. K = 1 tables only: the nearest atom's value is then exactly
// this chirp sum (hopping.cpp:92-99 with c = 1).
constexpr int kCpBins = 64;

__global__ void k_chirp_power(const float2* __restrict__ spec, int T, int P, int Mc, int M,
                              int tb, float* __restrict__ out) {
  extern __shared__ float pw[];  // [kCpBins][tb]
  const int batch = blockIdx.z, p = blockIdx.y, k0 = blockIdx.x * kCpBins;
  for (int e = threadIdx.x; e < kCpBins * tb; e += blockDim.x) {
    const int r = e / kCpBins, k = e % kCpBins;  // k fastest: coalesced reads
    const int t = batch * tb + r;
    float acc = 0.f;
    if (t < T && k0 + k < M) {
      const float2* z = spec + (((int64_t)t * P + p) * Mc) * M + k0 + k;
      for (int mc = 0; mc < Mc; ++mc) {
        const float2 v = z[(int64_t)mc * M];
        acc += v.x * v.x + v.y * v.y;
      }
    }
    pw[k * tb + r] = acc;
  }
  __syncthreads();
  float* dst = out + (((int64_t)batch * P + p) * M + k0) * tb;
  const int n = (M - k0 < kCpBins ? M - k0 : kCpBins) * tb;
  for (int e = threadIdx.x; e < n; e += blockDim.x) dst[e] = pw[e];
}

}  // namespace

void launch_chirp_power(Ctx* ctx, const float2* spec_d, int T, int P, int Mc, int M, int tb,
                        float* out_d) {
  const int n_tb = (T + tb - 1) / tb;
  if (n_tb > 65535) fail(GH_EINVAL, "spectra: too many trial batches for one launch");
  dim3 grid((M + kCpBins - 1) / kCpBins, P, n_tb);
  KTimer kt(ctx, "chirp_power");
  k_chirp_power<<<grid, 256, sizeof(float) * kCpBins * tb, ctx->stream>>>(spec_d, T, P, Mc, M, tb,
                                                                          out_d);
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

void launch_add_noise(Ctx* ctx, double2* frames_d, int T, int P, int N, uint64_t seed,
                      uint64_t trial0, double sigma) {
  const int64_t total = (int64_t)T * P * N;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148LL * 16));
  k_add_noise<<<blocks, 256, 0, ctx->stream>>>(frames_d, T, P, N, seed, trial0, sigma);
  GH_LAUNCHED(ctx);
}

}  // namespace gh
