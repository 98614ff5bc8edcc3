// gh_topk.cu — per-trial top-K local maxima of a decision map (sm_100a).
//
// BASELINE c3 (K = 5 targets, "top-5 local-maximum peak pick"): a bin is a
// local maximum if its value is > every lattice neighbour with a smaller
// index and >= every neighbour with a larger index (8 neighbours in 2-D, 26
// in 3-D; plateaus resolve to their smallest index, the argmax_index tie
// rule of src/direct.cpp:55-62). Candidates rank by (value desc, index asc).
// Restates oracle/gridhop_oracle.cpp or_topk_local_max.
//
// One CTA per trial. Each thread scans a strided set of bins, keeps its own
// top-K in registers and only tests the neighbourhood of bins that would
// enter that list (a pruning threshold), so the map is read ~once. The block
// then extracts the K best candidates with K block-wide argmax rounds.
#include <cuda_runtime.h>

#include "gh_internal.cuh"

namespace gh {
namespace {

constexpr int kTopkThreads = 256;
constexpr int kMaxK = 8;

__device__ __forceinline__ bool better(float v, int64_t i, float bv, int64_t bi) {
  return v > bv || (v == bv && i < bi);
}

__global__ void __launch_bounds__(kTopkThreads) k_topk_localmax(const float* __restrict__ map,
                                                               int64_t G, int nx, int ny, int nz,
                                                               int K, int64_t bin0, int64_t* idx_out,
                                                               float* val_out) {
  const int trial = blockIdx.x;
  const float* m = map + (int64_t)trial * G;
  // sorted (value desc, index asc); empty slots are (-inf, INT64_MAX). Only
  // compile-time indices touch tv/ti so they stay in registers.
  float tv[kMaxK];
  int64_t ti[kMaxK];
#pragma unroll
  for (int k = 0; k < kMaxK; ++k) {
    tv[k] = -INFINITY;
    ti[k] = INT64_MAX;
  }
  const int64_t nxy = (int64_t)nx * ny;
  for (int64_t i = threadIdx.x; i < G; i += kTopkThreads) {
    const float v = m[i];
    float lastv = tv[0];
    int64_t lasti = ti[0];
#pragma unroll
    for (int k = 1; k < kMaxK; ++k)
      if (k == K - 1) {
        lastv = tv[k];
        lasti = ti[k];
      }
    // prune: cannot enter this thread's top-K
    if (!better(v, i, lastv, lasti)) continue;
    const int64_t x = i % nx, y = (i / nx) % ny, z = i / nxy;
    bool ok = true;
    for (int dz = -1; dz <= 1 && ok; ++dz) {
      const int64_t zz = z + dz;
      if (zz < 0 || zz >= nz) continue;
      for (int dy = -1; dy <= 1 && ok; ++dy) {
        const int64_t yy = y + dy;
        if (yy < 0 || yy >= ny) continue;
        for (int dx = -1; dx <= 1 && ok; ++dx) {
          if (!dx && !dy && !dz) continue;
          const int64_t xx = x + dx;
          if (xx < 0 || xx >= nx) continue;
          const int64_t j = (zz * ny + yy) * nx + xx;
          const float w = m[j];
          ok = (j < i) ? (v > w) : (v >= w);
        }
      }
    }
    if (!ok) continue;
    // insertion from the bottom (slot K-1 is known to be displaced)
    bool done = false;
#pragma unroll
    for (int k = kMaxK - 1; k >= 0; --k) {
      if (k < K && !done) {
        if (k > 0 && better(v, i, tv[k - 1], ti[k - 1])) {
          tv[k] = tv[k - 1];
          ti[k] = ti[k - 1];
        } else {
          tv[k] = v;
          ti[k] = i;
          done = true;
        }
      }
    }
  }
  // block-wide K rounds of argmax over the per-thread heads
  __shared__ float sv[kTopkThreads / 32];
  __shared__ int64_t si[kTopkThreads / 32];
  __shared__ int sw[kTopkThreads / 32];
  __shared__ int winner;
  int head = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < K; ++k) {
    float v = -INFINITY;
    int64_t i = INT64_MAX;
#pragma unroll
    for (int s = 0; s < kMaxK; ++s)
      if (s == head && s < K) {
        v = tv[s];
        i = ti[s];
      }
    int who = threadIdx.x;
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, i, o);
      const int ow = __shfl_xor_sync(0xffffffffu, who, o);
      if (better(ov, oi, v, i)) {
        v = ov;
        i = oi;
        who = ow;
      }
    }
    if (lane == 0) {
      sv[warp] = v;
      si[warp] = i;
      sw[warp] = who;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float bv = sv[0];
      int64_t bi = si[0];
      int bw = sw[0];
      for (int w = 1; w < kTopkThreads / 32; ++w)
        if (better(sv[w], si[w], bv, bi)) {
          bv = sv[w];
          bi = si[w];
          bw = sw[w];
        }
      const bool valid = bi != INT64_MAX && bv != -INFINITY;
      idx_out[(int64_t)trial * K + k] = valid ? bin0 + bi : -1;
      val_out[(int64_t)trial * K + k] = valid ? bv : 0.0f;
      winner = valid ? bw : -1;
    }
    __syncthreads();
    if (threadIdx.x == winner) ++head;
    __syncthreads();
  }
}

}  // namespace

void launch_topk(Ctx* ctx, const float* map_d, int T, const gh_grid& g, int K, int64_t bin0,
                 int64_t* idx_d,
                 float* val_d) {
  if (K < 1 || K > kMaxK) fail(GH_EINVAL, "top-k: k must be in [1, 8]");
  const int64_t G = (int64_t)g.n[0] * g.n[1] * g.n[2];
  KTimer kt(ctx, "topk");
  k_topk_localmax<<<T, kTopkThreads, 0, ctx->stream>>>(map_d, G, g.n[0], g.n[1], g.n[2], K, bin0, idx_d,
                                                       val_d);
  GH_LAUNCHED(ctx);
}

}  // namespace gh
