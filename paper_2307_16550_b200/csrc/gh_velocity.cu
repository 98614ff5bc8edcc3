// gh_velocity.cu — the velocity stage after the location peak (sm_100a).
//
// Reference: hop_velocity (src/hopping.cpp:185-236) and direct_velocity +
// velocity_stage / velocity_value (src/direct.cpp:145-228); SURVEY §8f rank
// 1. Batched over trials at their located bins, on multi-chirp frames
// [T][P][Mc][N]:
//   k_vel_stage    one CTA per (trial, pair): x_hat from the located bin
//                  (fp64, bit-identical grid point and sensed range), the
//                  conjugate range atom in shared memory, range compression
//                  h[m] = sum_n y[m][n] conj(a(r))[n] with a warp per chirp,
//                  and the Doppler direction sum doppler_scale*(u_tx + u_rx);
//   hop:           the zero-padded slow-time spectra of h (the range-FFT
//                  kernel with N = Mc, os = os_doppler), then k_hop_vel_scan:
//                  one CTA per trial scans the velocity grid, each point
//                  summing the pairs' power at lround(dir . v * os_d) mod n_d;
//   direct:        k_direct_vel: one CTA per trial, each velocity point
//                  correlating h with the conjugate Doppler atom of every pair
//                  (fp32 phasor recurrence re-seeded from fp64 every 32
//                  chirps);
// both keep the first maximum (VelocityGrid order, ties to the smaller
// index), as the reference's scans do.
#include <cuda_runtime.h>

#include <algorithm>

#include "gh_internal.cuh"

namespace gh {
namespace {

constexpr int kVsThreads = 256;

__global__ void __launch_bounds__(kVsThreads) k_vel_stage(const float2* __restrict__ frames, int P,
                                                          int Mc, int N,
                                                          const double* __restrict__ txrx,
                                                          gh_grid grid, double scale,
                                                          double doppler_scale,
                                                          const int64_t* __restrict__ loc,
                                                          float2* __restrict__ h,
                                                          double* __restrict__ dirs) {
  extern __shared__ float2 ca[];  // conj(a(r))[n], n < N
  const int t = blockIdx.x / P, p = blockIdx.x % P;
  double x[3];
  dgrid_point(grid, loc[t], x);
  const double* tx = txrx + 6 * p;
  const double* rx = tx + 3;
  const double dtx = dnorm3(tx, x[0], x[1], x[2]);
  const double drx = dnorm3(rx, x[0], x[1], x[2]);
  const double r = __dmul_rn(scale, __dadd_rn(dtx, drx));
  const double rho = r / (double)N;  // turns per sample
  for (int n = threadIdx.x; n < N; n += kVsThreads) {
    const double ph = rho * (double)n;
    float s, c;
    sincospif((float)(2.0 * (ph - floor(ph))), &s, &c);
    ca[n] = make_float2(c, -s);
  }
  if (threadIdx.x == 0) {
    for (int d = 0; d < 3; ++d)
      dirs[((int64_t)t * P + p) * 3 + d] =
          doppler_scale * ((x[d] - tx[d]) / dtx + (x[d] - rx[d]) / drx);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float2* y = frames + (((int64_t)t * P + p) * Mc) * N;
  for (int m = warp; m < Mc; m += kVsThreads / 32) {
    float re = 0.f, im = 0.f;
    for (int n = lane; n < N; n += 32) {
      const float2 v = y[(int64_t)m * N + n], w = ca[n];
      re += v.x * w.x - v.y * w.y;
      im += v.x * w.y + v.y * w.x;
    }
    for (int o = 16; o > 0; o >>= 1) {
      re += __shfl_xor_sync(0xffffffffu, re, o);
      im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    if (lane == 0) h[((int64_t)t * P + p) * Mc + m] = make_float2(re, im);
  }
}

// block-wide first maximum over (value, index): larger value, then smaller index
__device__ __forceinline__ void block_argmax(float& v, int64_t& k, float* sv, int64_t* sk) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t ok = __shfl_xor_sync(0xffffffffu, k, o);
    if (ok >= 0 && (k < 0 || ov > v || (ov == v && ok < k))) {
      v = ov;
      k = ok;
    }
  }
  if (lane == 0) {
    sv[warp] = v;
    sk[warp] = k;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x / 32); ++w)
      if (sk[w] >= 0 && (k < 0 || sv[w] > v || (sv[w] == v && sk[w] < k))) {
        v = sv[w];
        k = sk[w];
      }
  }
}

__device__ __forceinline__ void velocity_point(double spacing, int half, int64_t k, double* v) {
  const int64_t n = 2 * (int64_t)half + 1;
  v[0] = spacing * (double)(k % n - half);
  v[1] = spacing * (double)(k / n - half);
}

__global__ void __launch_bounds__(kVsThreads) k_hop_vel_scan(const float2* __restrict__ dspec,
                                                             const double* __restrict__ dirs,
                                                             int P, int nd, int os_d,
                                                             double spacing, int half,
                                                             int64_t* __restrict__ vidx,
                                                             float* __restrict__ vval) {
  __shared__ float sv[kVsThreads / 32];
  __shared__ int64_t sk[kVsThreads / 32];
  const int t = blockIdx.x;
  const int64_t V = (2 * (int64_t)half + 1) * (2 * (int64_t)half + 1);
  const float2* sp = dspec + (int64_t)t * P * nd;
  const double* dr = dirs + (int64_t)t * P * 3;
  float best = -1.f;
  int64_t bk = -1;
  for (int64_t k = threadIdx.x; k < V; k += kVsThreads) {  // ascending per thread
    double v[2];
    velocity_point(spacing, half, k, v);
    float value = 0.f;
    for (int q = 0; q < P; ++q) {
      const double u = __dadd_rn(__dmul_rn(dr[3 * q], v[0]), __dmul_rn(dr[3 * q + 1], v[1]));
      const long long bin = llround(u * (double)os_d);
      const int idx = (int)(((bin % nd) + nd) % nd);
      const float2 z = sp[(int64_t)q * nd + idx];
      value += z.x * z.x + z.y * z.y;
    }
    if (value > best) {
      best = value;
      bk = k;
    }
  }
  block_argmax(best, bk, sv, sk);
  if (threadIdx.x == 0) {
    vidx[t] = bk;
    vval[t] = best;
  }
}

__global__ void __launch_bounds__(kVsThreads) k_direct_vel(const float2* __restrict__ h,
                                                           const double* __restrict__ dirs, int P,
                                                           int Mc, double spacing, int half,
                                                           int64_t* __restrict__ vidx,
                                                           float* __restrict__ vval) {
  extern __shared__ float2 hs[];  // [P][Mc]
  __shared__ float sv[kVsThreads / 32];
  __shared__ int64_t sk[kVsThreads / 32];
  const int t = blockIdx.x;
  for (int e = threadIdx.x; e < P * Mc; e += kVsThreads) hs[e] = h[(int64_t)t * P * Mc + e];
  __syncthreads();
  const int64_t V = (2 * (int64_t)half + 1) * (2 * (int64_t)half + 1);
  const double* dr = dirs + (int64_t)t * P * 3;
  float best = -1.f;
  int64_t bk = -1;
  for (int64_t k = threadIdx.x; k < V; k += kVsThreads) {
    double v[2];
    velocity_point(spacing, half, k, v);
    float value = 0.f;
    for (int q = 0; q < P; ++q) {
      const double u = __dadd_rn(__dmul_rn(dr[3 * q], v[0]), __dmul_rn(dr[3 * q + 1], v[1]));
      const double rho = u / (double)Mc;  // turns per chirp
      float sw, cw;
      sincospif((float)(2.0 * (rho - floor(rho))), &sw, &cw);
      float zr = 0.f, zi = 0.f, pr = 1.f, pi = 0.f;
      for (int m = 0; m < Mc; ++m) {
        if ((m & 31) == 0 && m) {  // re-seed: exact phase every 32 chirps
          const double ph = rho * (double)m;
          float s, c;
          sincospif((float)(2.0 * (ph - floor(ph))), &s, &c);
          pr = c;
          pi = s;
        }
        // conj(b(u))[m] = exp(-j 2 pi u m / Mc) = (pr, -pi)
        const float2 hm = hs[q * Mc + m];
        zr += hm.x * pr + hm.y * pi;
        zi += hm.y * pr - hm.x * pi;
        const float nr = pr * cw - pi * sw;
        pi = pr * sw + pi * cw;
        pr = nr;
      }
      value += zr * zr + zi * zi;
    }
    if (value > best) {
      best = value;
      bk = k;
    }
  }
  block_argmax(best, bk, sv, sk);
  if (threadIdx.x == 0) {
    vidx[t] = bk;
    vval[t] = best;
  }
}

}  // namespace

void launch_velocity(Ctx* ctx, const double* txrx_d, const gh_wave* w, const gh_grid* g,
                     const gh_velocity_grid* vg, const float2* frames_d, int T, int Mc,
                     const int64_t* loc_d, bool hop, int64_t* vidx_d, float* vval_d) {
  const int P = w->n_pairs, N = w->n_samples;
  const int nd = vg->os_doppler * Mc;
  // scratch: h [T][P][Mc] complex64, dirs [T][P][3] fp64, Doppler spectra
  const size_t h_bytes = sizeof(float2) * (size_t)T * P * Mc;
  const size_t d_bytes = sizeof(double) * (size_t)T * P * 3;
  const size_t s_bytes = hop ? sizeof(float2) * (size_t)T * P * nd : 0;
  auto* base = static_cast<unsigned char*>(ctx->misc2.get(h_bytes + d_bytes + s_bytes));
  auto* h = reinterpret_cast<float2*>(base);
  auto* dirs = reinterpret_cast<double*>(base + h_bytes);
  auto* dspec = reinterpret_cast<float2*>(base + h_bytes + d_bytes);
  {
    KTimer kt(ctx, "vel_stage");
    const int64_t blocks = (int64_t)T * P;
    if (blocks > 0x7fffffff) fail(GH_EINVAL, "velocity: too many trials");
    k_vel_stage<<<static_cast<unsigned>(blocks), kVsThreads, sizeof(float2) * N, ctx->stream>>>(
        frames_d, P, Mc, N, txrx_d, *g, w->range_scale, vg->doppler_scale, loc_d, h, dirs);
    GH_LAUNCHED(ctx);
  }
  if (hop) {
    // zero-padded slow-time spectra of h: n_d = os_doppler * Mc points
    launch_fft(ctx, h, nullptr, T, P, Mc, vg->os_doppler, 16, FFT_NATURAL, dspec);
    KTimer kt(ctx, "vel_scan");
    k_hop_vel_scan<<<T, kVsThreads, 0, ctx->stream>>>(dspec, dirs, P, nd, vg->os_doppler,
                                                      vg->spacing, vg->half, vidx_d, vval_d);
    GH_LAUNCHED(ctx);
  } else {
    const size_t smem = sizeof(float2) * (size_t)P * Mc;
    if (smem > 200 * 1024) fail(GH_EINVAL, "velocity: too many pairs x chirps");
    GH_CUDA(cudaFuncSetAttribute(k_direct_vel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    KTimer kt(ctx, "vel_scan");
    k_direct_vel<<<T, kVsThreads, smem, ctx->stream>>>(h, dirs, P, Mc, vg->spacing, vg->half,
                                                       vidx_d, vval_d);
    GH_LAUNCHED(ctx);
  }
}

}  // namespace gh
