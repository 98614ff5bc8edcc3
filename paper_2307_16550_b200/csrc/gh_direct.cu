// gh_direct.cu — the direct method (exhaustive location correlation).
//
// Reference: location_decision_map (src/direct.cpp:90-144) and conj_atom
// (src/direct.cpp:20-35), Mc = 1:
//   value(bin) = sum_p | sum_n y_p[n] conj(a_n(r_p(bin))) |^2,
//   a_n(r) = exp(j 2pi r n / N)
// computed for T trials at once as the complex contraction
//   Z_p (T x G) = Y_p (T x N) . A_p^H (N x G),
// |Z_p|^2 summed over pairs in the epilogue, then per-trial argmax (the
// argmax_index tie rule) through the same 64-bit key as the gather.
//
// This file holds the CUDA-core (SIMT fp32) contraction: 64 trials x 64 bins
// per CTA, the steering tile generated on the fly (phase reduced in fp64,
// fp32 sincospi). It is the correctness path and the baseline for the
// tcgen05 kernel in gh_direct_umma.cu.
#include <cuda_runtime.h>

#include "gh_internal.cuh"

namespace gh {
namespace {

constexpr int BT = 64, BG = 64, BN = 32;

struct DirectArgs {
  const float2* frames;  // [T][P][N]
  const double* txrx;    // [P][6]
  gh_grid grid;
  double scale;
  int T, P, N;
  int64_t G;
  int mag;
  float* map;
  unsigned long long* keys;
};

__global__ void __launch_bounds__(256) k_direct_simt(DirectArgs a) {
  __shared__ float2 ys[BN][BT];
  __shared__ float2 as[BN][BG];
  __shared__ double rr[BG];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int t0 = blockIdx.x * BT;
  const int64_t g0 = (int64_t)blockIdx.y * BG;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const double inv_n = 1.0 / (double)a.N;
  for (int p = 0; p < a.P; ++p) {
    __syncthreads();
    if (threadIdx.x < BG) {
      const int64_t g = g0 + threadIdx.x;
      double r = 0.0;
      if (g < a.G) {
        double x[3];
        dgrid_point(a.grid, g, x);
        const double* tp = a.txrx + 6 * p;
        r = __dmul_rn(a.scale, __dadd_rn(dnorm3(tp, x[0], x[1], x[2]), dnorm3(tp + 3, x[0], x[1], x[2])));
      }
      rr[threadIdx.x] = r * inv_n;  // turns per sample
    }
    float zr[4][4], zi[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) zr[i][j] = zi[i][j] = 0.f;
    for (int n0 = 0; n0 < a.N; n0 += BN) {
      __syncthreads();
      for (int e = threadIdx.x; e < BN * BT; e += 256) {
        const int n = e / BT, t = e % BT;
        const int tt = t0 + t;
        ys[n][t] = (tt < a.T && n0 + n < a.N)
                       ? a.frames[((int64_t)tt * a.P + p) * a.N + n0 + n]
                       : make_float2(0.f, 0.f);
      }
      for (int e = threadIdx.x; e < BN * BG; e += 256) {
        const int n = e / BG, g = e % BG;
        const double ph = rr[g] * (double)(n0 + n);
        const double fr = ph - floor(ph);
        float s, c;
        sincospif((float)(2.0 * fr), &s, &c);
        as[n][g] = (n0 + n < a.N) ? make_float2(c, s) : make_float2(0.f, 0.f);
      }
      __syncthreads();
#pragma unroll 8
      for (int n = 0; n < BN; ++n) {
        float2 y[4], w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) y[i] = ys[n][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = as[n][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            // y * conj(a)
            zr[i][j] += y[i].x * w[j].x + y[i].y * w[j].y;
            zi[i][j] += y[i].y * w[j].x - y[i].x * w[j].y;
          }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float pw = zr[i][j] * zr[i][j] + zi[i][j] * zi[i][j];
        acc[i][j] += a.mag ? sqrtf(pw) : pw;
      }
  }
  if (a.map) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int t = t0 + ty + 16 * i;
      if (t >= a.T) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t g = g0 + tx + 16 * j;
        if (g < a.G) a.map[(int64_t)t * a.G + g] = acc[i][j];
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float bv = -1.f;
    int bg = -1;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t g = g0 + tx + 16 * j;
      if (g < a.G && acc[i][j] > bv) {
        bv = acc[i][j];
        bg = tx + 16 * j;
      }
    }
    for (int o = 1; o < 16; o <<= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int og = __shfl_xor_sync(0xffffffffu, bg, o);
      if (og >= 0 && (ov > bv || (ov == bv && og < bg))) {
        bv = ov;
        bg = og;
      }
    }
    const int t = t0 + ty + 16 * i;
    if (tx == 0 && t < a.T && bg >= 0) {
      const unsigned long long gb = (unsigned long long)(g0 + bg);
      atomicMax(a.keys + t, ((unsigned long long)__float_as_uint(bv) << 32) | (0xffffffffull - gb));
    }
  }
}

}  // namespace

void direct_map_simt(Ctx* ctx, const double* txrx_d, const gh_wave* w, const gh_grid* g,
                     const float2* frames_d, int T, int combine, float* map_d,
                     unsigned long long* keys_d) {
  DirectArgs a{};
  a.frames = frames_d;
  a.txrx = txrx_d;
  a.grid = *g;
  a.scale = w->range_scale;
  a.T = T;
  a.P = w->n_pairs;
  a.N = w->n_samples;
  a.G = (int64_t)g->n[0] * g->n[1] * g->n[2];
  a.mag = combine == GH_MAGNITUDE;
  a.map = map_d;
  a.keys = keys_d;
  const int64_t gb = (a.G + BG - 1) / BG;
  if (gb > 65535) fail(GH_EINVAL, "direct: grid too large for the SIMT path");
  dim3 grid((T + BT - 1) / BT, static_cast<unsigned>(gb));
  KTimer kt(ctx, "direct_simt");
  k_direct_simt<<<grid, 256, 0, ctx->stream>>>(a);
  GH_LAUNCHED(ctx);
}

}  // namespace gh
