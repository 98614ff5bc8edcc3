// gh_fft.cu — beat-signal synthesis and the zero-padded range FFT (sm_100a).
//
// Reference: fast_time_spectra / fft_rows (src/hopping.cpp:121-129,
// src/fft.cpp:132-146, include/gridhop/fft.hpp:7-10): out[i] =
// sum_n y[n] exp(-j 2pi i n / M), M = os * N, forward and unnormalised.
// Synthesis restates synthesize_frame + add_noise (src/synth.cpp:15-49) and
// sample_scene (src/montecarlo.cpp:48-66) on the counter-based stream shared
// with the oracle.
//
// One CTA owns TB trials of one pair (blockIdx = (trial batch, pair)) and
// transforms them R rows at a time in shared memory:
//   * zero padding is pruned: with bit-reversed input order the N non-zero
//     samples land on multiples of os, and the first log2(os) DIT stages of
//     a block (y, 0, .., 0) just replicate y, so the load writes each sample
//     os times and the butterflies start at half = os;
//   * the epilogue writes the gather layout [batch][pair][M][TB] (one
//     contiguous TB-run per range bin, TB = trials of the batch) as power,
//     magnitude or complex, or the natural [T][P][M] layout for parity.
// Row pitch (M + 16/R float2) makes the transposing epilogue reads
// bank-conflict free.
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

struct FftArgs {
  const float2* frames;  // [T][P][N] (or null with synth)
  SynthParams sp;
  int synth;
  int T, P, N, M, log2n, log2m, log2os, os;
  int tb, rows, log2rows, pitch;
  int out_kind;
  const float2* tw;      // exp(-2 pi i k / M), k < M/2
  void* out;
};

__global__ void __launch_bounds__(kFftThreads, 1) k_fft(FftArgs a) {
  extern __shared__ float2 sm[];
  __shared__ RowSynth rsm[16];
  const int tb = blockIdx.x, p = blockIdx.y;
  const int R = a.rows, M = a.M, N = a.N;
  const int halfM = M >> 1;
  const double inv_n = 1.0 / (double)N;
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
    // load: bit-reversed, each sample replicated over its os-block
    for (int e = threadIdx.x; e < R * N; e += blockDim.x) {
      const int r = e >> a.log2n;
      const int g = e & (N - 1);
      const int n = a.log2n ? (int)(__brev((unsigned)g) >> (32 - a.log2n)) : 0;
      const int t = tb * a.tb + g0 + r;
      float2 v = make_float2(0.f, 0.f);
      if (t < a.T) {
        if (a.synth)
          v = synth_sample(rsm[r], a.sp.camp.n_targets, n, inv_n);
        else
          v = a.frames[((int64_t)t * a.P + p) * N + n];
      }
      float2* dst = sm + r * a.pitch + (g << a.log2os);
      for (int j = 0; j < a.os; ++j) dst[j] = v;
    }
    __syncthreads();
    // radix-2 DIT stages from half = os
    for (int half = a.os, lh = a.log2os; half < M; half <<= 1, ++lh) {
      const int tw_step = halfM >> lh;  // M / (2 half)
      for (int e = threadIdx.x; e < R * halfM; e += blockDim.x) {
        const int r = e >> (a.log2m - 1);
        const int b = e & (halfM - 1);
        const int j = b & (half - 1);
        const int i0 = ((b >> lh) << (lh + 1)) + j;
        float2* x = sm + r * a.pitch;
        const float2 w = __ldg(a.tw + j * tw_step);
        const float2 u = x[i0], v0 = x[i0 + half];
        const float2 v = make_float2(v0.x * w.x - v0.y * w.y, v0.x * w.y + v0.y * w.x);
        x[i0] = make_float2(u.x + v.x, u.y + v.y);
        x[i0 + half] = make_float2(u.x - v.x, u.y - v.y);
      }
      __syncthreads();
    }
    // epilogue
    if (a.out_kind == FFT_NATURAL) {
      float2* out = static_cast<float2*>(a.out);
      for (int e = threadIdx.x; e < R * M; e += blockDim.x) {
        const int r = e >> a.log2m, i = e & (M - 1);
        const int t = tb * a.tb + g0 + r;
        if (t < a.T) out[((int64_t)t * a.P + p) * M + i] = sm[r * a.pitch + i];
      }
    } else {
      const int64_t base = ((int64_t)tb * a.P + p) * M;
      for (int e = threadIdx.x; e < R * M; e += blockDim.x) {
        const int i = e >> a.log2rows, r = e & (R - 1);
        const float2 z = sm[r * a.pitch + i];
        const int64_t o = (base + i) * a.tb + g0 + r;
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

int ilog2(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}

const float2* twiddles(Ctx* ctx, int M) {
  if (ctx->twiddle_m != M) {
    std::vector<float2> h(static_cast<size_t>(M / 2));
    for (int k = 0; k < M / 2; ++k) {
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
  if (M > 65536) fail(GH_EINVAL, "spectra: FFT length above 65536 unsupported");
  if (tb < 1 || tb > 32 || (tb & (tb - 1))) fail(GH_EINVAL, "spectra: bad trial batch");
  FftArgs a{};
  a.frames = frames_d;
  a.synth = synth != nullptr;
  if (synth) a.sp = *synth;
  a.T = T;
  a.P = P;
  a.N = N;
  a.M = M;
  a.log2n = ilog2(N);
  a.log2m = ilog2(M);
  a.os = os;
  a.log2os = ilog2(os);
  a.tb = tb;
  // rows per pass: power of two <= min(tb, 16) within ~200 KB of smem
  int R = tb < 16 ? tb : 16;
  while (R > 1 && static_cast<size_t>(R) * (M + 16) * sizeof(float2) > 200 * 1024) R >>= 1;
  a.rows = R;
  a.log2rows = ilog2(R);
  a.pitch = M + 16 / (R < 16 ? R : 16);
  a.out_kind = out_kind;
  a.tw = twiddles(ctx, M);
  a.out = out_d;
  const size_t smem = static_cast<size_t>(R) * a.pitch * sizeof(float2);
  GH_CUDA(cudaFuncSetAttribute(k_fft, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  const int n_tb = (T + tb - 1) / tb;
  dim3 grid(n_tb, P);
  KTimer kt(ctx, synth ? "synth_fft" : "fft");
  k_fft<<<grid, kFftThreads, smem, ctx->stream>>>(a);
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
