// gh_indirect.cu — the indirect pipeline's location stage (sm_100a).
//
// Reference: range_doppler_map + RangeDopplerMap::peak + multilaterate_location
// (src/indirect.cpp:10-83). At Mc = 1 (the BASELINE
// frames) a receiver's range-Doppler map is the modulus of its zero-padded
// range spectrum; its peak (first maximum) gives r_hat = bin / os_range, and
// the location is the grid bin minimising sum_q (sensed_range(x) - r_hat_q)^2
// (first minimum).
//
// k_range_peaks: one warp per (trial, pair) spectrum row, running first-max
// of |Z|^2 per lane, then a shuffle merge (larger value, then smaller bin).
// k_multilat: CTA = (bin chunk, batch of trials); the chunk's sensed ranges
// (fp64, [P][chunk]) are staged in shared memory and every trial of the
// batch scans them. The residual is evaluated exactly as the reference does
// (d = r - r_hat, res += d * d, pairs ascending, each operation rounded: no
// FMA), so the GPU and the -ffp-contract=off oracle agree bit for bit.
// Per (trial, chunk) winners merge in k_multilat_reduce.
#include <cuda_runtime.h>

#include <algorithm>

#include "gh_internal.cuh"

namespace gh {
namespace {

constexpr int kMlThreads = 256;
constexpr int kMlTrials = 32;   // trials per CTA
constexpr int kMlParts = kMlThreads / kMlTrials;  // threads per trial
constexpr int kMlChunk = 256;   // bins per CTA

__global__ void k_range_peaks(const float2* __restrict__ spec, int64_t rows, int M, int os,
                              double* __restrict__ rhat) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;  // whole warps
  const float2* z = spec + row * M;
  float best = -1.f;
  int bk = 0;
  for (int k = lane; k < M; k += 32) {
    const float2 v = z[k];
    const float p = v.x * v.x + v.y * v.y;
    if (p > best) {
      best = p;
      bk = k;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
    if (ob > best || (ob == best && ok < bk)) {
      best = ob;
      bk = ok;
    }
  }
  if (lane == 0) rhat[row] = (double)bk / (double)os;
}

// sensed ranges of every (pair, bin), fp64, [P][G] (a1, model.cpp:45-52)
__global__ void k_ranges(const double* __restrict__ txrx, gh_grid grid, double scale, int P,
                         int64_t G, double* __restrict__ r) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)P * G;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(e / G);
    const int64_t g = e - (int64_t)p * G;
    double x[3];
    dgrid_point(grid, g, x);
    const double* tp = txrx + 6 * p;
    r[e] = __dmul_rn(scale, __dadd_rn(dnorm3(tp, x[0], x[1], x[2]), dnorm3(tp + 3, x[0], x[1], x[2])));
  }
}

__global__ void __launch_bounds__(kMlThreads) k_multilat(const double* __restrict__ r, int P,
                                                         int64_t G, const double* __restrict__ rhat,
                                                         int T, double* __restrict__ cand_res,
                                                         int64_t* __restrict__ cand_idx) {
  extern __shared__ double sr[];              // [P][kMlChunk] sensed ranges of the chunk
  double* srh = sr + (size_t)P * kMlChunk;    // [kMlTrials][P] r_hat of the batch
  const int64_t g0 = (int64_t)blockIdx.x * kMlChunk;
  const int t0 = blockIdx.y * kMlTrials;
  const int nb = (int)std::min<int64_t>(kMlChunk, G - g0);
  for (int e = threadIdx.x; e < P * kMlChunk; e += kMlThreads) {
    const int p = e / kMlChunk, b = e % kMlChunk;
    sr[e] = b < nb ? r[(int64_t)p * G + g0 + b] : 0.0;
  }
  for (int e = threadIdx.x; e < kMlTrials * P; e += kMlThreads) {
    const int t = t0 + e / P;
    srh[e] = t < T ? rhat[(int64_t)t0 * P + e] : 0.0;
  }
  __syncthreads();
  const int tl = threadIdx.x / kMlParts, part = threadIdx.x % kMlParts;
  const double* rh = srh + tl * P;
  double best = -1.0;
  int bb = 0;
  for (int b = part; b < nb; b += kMlParts) {  // ascending bins per thread
    double res = 0.0;
    for (int p = 0; p < P; ++p) {
      const double d = __dsub_rn(sr[p * kMlChunk + b], rh[p]);
      res = __dadd_rn(res, __dmul_rn(d, d));
    }
    if (best < 0.0 || res < best) {
      best = res;
      bb = b;
    }
  }
  // merge the kMlParts threads of this trial: smaller residual, then smaller bin
  for (int o = kMlParts / 2; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int obb = __shfl_xor_sync(0xffffffffu, bb, o);
    if (ob >= 0.0 && (best < 0.0 || ob < best || (ob == best && obb < bb))) {
      best = ob;
      bb = obb;
    }
  }
  const int t = t0 + tl;
  if (part == 0 && t < T) {
    cand_res[(int64_t)t * gridDim.x + blockIdx.x] = best;
    cand_idx[(int64_t)t * gridDim.x + blockIdx.x] = g0 + bb;
  }
}

// per trial: the first minimum over the chunk winners (chunks ascend in bin)
__global__ void k_multilat_reduce(const double* __restrict__ cand_res,
                                  const int64_t* __restrict__ cand_idx, int T, int n_chunks,
                                  int64_t* __restrict__ idx, double* __restrict__ res) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  double best = -1.0;
  int64_t bi = 0;
  for (int c = 0; c < n_chunks; ++c) {
    const double v = cand_res[(int64_t)t * n_chunks + c];
    if (best < 0.0 || v < best) {
      best = v;
      bi = cand_idx[(int64_t)t * n_chunks + c];
    }
  }
  idx[t] = bi;
  res[t] = best;
}

}  // namespace

void launch_range_peaks(Ctx* ctx, const float2* spec_d, int64_t rows, int M, int os,
                        double* rhat_d) {
  KTimer kt(ctx, "range_peaks");
  const int64_t threads = rows * 32;
  k_range_peaks<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, ctx->stream>>>(
      spec_d, rows, M, os, rhat_d);
  GH_LAUNCHED(ctx);
}

void launch_multilaterate(Ctx* ctx, const double* txrx_d, const gh_wave* w, const gh_grid* g,
                          const double* rhat_d, int T, int64_t* idx_d, double* res_d) {
  const int P = w->n_pairs;
  const int64_t G = (int64_t)g->n[0] * g->n[1] * g->n[2];
  const int64_t n_chunks = (G + kMlChunk - 1) / kMlChunk;
  if (n_chunks > 0x7fffffff) fail(GH_EINVAL, "multilateration: grid too large");
  const int n_tb = (T + kMlTrials - 1) / kMlTrials;
  if (n_tb > 65535) fail(GH_EINVAL, "multilateration: too many trials for one launch");
  const size_t smem = sizeof(double) * ((size_t)P * kMlChunk + (size_t)kMlTrials * P);
  if (smem > 200 * 1024) fail(GH_EINVAL, "multilateration: too many pairs");
  // scratch: sensed ranges [P][G], then the per-(trial, chunk) winners
  const size_t r_bytes = sizeof(double) * P * G;
  const size_t c_bytes = (sizeof(double) + sizeof(int64_t)) * (size_t)T * n_chunks;
  auto* base = static_cast<unsigned char*>(ctx->misc2.get(r_bytes + c_bytes));
  auto* r = reinterpret_cast<double*>(base);
  auto* cres = reinterpret_cast<double*>(base + r_bytes);
  auto* cidx = reinterpret_cast<int64_t*>(cres + (size_t)T * n_chunks);
  {
    KTimer kt(ctx, "ranges");
    const int blocks = static_cast<int>(std::min<int64_t>((P * G + 255) / 256, 148LL * 16));
    k_ranges<<<blocks, 256, 0, ctx->stream>>>(txrx_d, *g, w->range_scale, P, G, r);
    GH_LAUNCHED(ctx);
  }
  {
    KTimer kt(ctx, "multilaterate");
    GH_CUDA(cudaFuncSetAttribute(k_multilat, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    k_multilat<<<dim3(static_cast<unsigned>(n_chunks), n_tb), kMlThreads, smem, ctx->stream>>>(
        r, P, G, rhat_d, T, cres, cidx);
    GH_LAUNCHED(ctx);
    k_multilat_reduce<<<(T + 255) / 256, 256, 0, ctx->stream>>>(cres, cidx, T,
                                                                static_cast<int>(n_chunks), idx_d,
                                                                res_d);
    GH_LAUNCHED(ctx);
  }
}

}  // namespace gh
