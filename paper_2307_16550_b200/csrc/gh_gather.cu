// gh_gather.cu — the grid-hopping gather-accumulate with fused argmax
// (sm_100a).
//
// Reference: hop_bin_value / scan_planes (src/hopping.cpp:59-117):
//   value(bin) = sum_q | sum_j c_j Z_q[I_j(bin, q)] |^2
// with Mc = 1, and argmax_index (src/direct.cpp:55-62, first strict max).
//
// One CTA = (trial batch of TB trials, location tile). It stages the tile's
// per-pair range windows of the batch's spectra into shared memory (layout
// [row][trial], one TB-run per row, so the TB lanes of a bin read one
// contiguous, bank-conflict-free run), then every warp walks bins: lane t
// of a TB-lane group accumulates trial t's value for one bin over all
// pairs. The table (uint16 shared-memory rows, 4 pairs per 64-bit load) is
// read once per batch of TB trials and broadcast within the lane group.
// Argmax is fused: per-thread running max over its bins (increasing order,
// strict >), merged across warps with the smallest-index tie rule, then one
// 64-bit atomicMax per (CTA, trial) on key = float_bits(value) << 32 |
// (2^32 - 1 - bin), which orders by value and then by smallest bin.
#include <cuda_runtime.h>

#include "gh_internal.cuh"

namespace gh {
namespace {

constexpr int kGatherThreads = 512;

struct GatherArgs {
  const void* spec;       // [batches][P][M][TB] float or float2
  const TileDesc* tiles;  // tiled plan
  const int4* win;        // [tiles][P] / [P]
  const uint16_t* rows;   // [entries][p4]
  const float2* coef3;    // [entries][P][3]
  gh_grid grid;
  int64_t G;
  int64_t chunk_bins;     // full plan
  int full;
  int P, p4, M, T;
  float* map;             // parity mode [T][G]
  unsigned long long* keys;
};

template <int TB, bool K3, bool MAG, bool MAPMODE>
__global__ void __launch_bounds__(kGatherThreads, 1) k_gather(GatherArgs a) {
  using E = typename std::conditional<K3, float2, float>::type;
  extern __shared__ __align__(16) unsigned char smraw[];
  E* sm = reinterpret_cast<E*>(smraw);
  constexpr int BPW = 32 / TB;  // bins per warp step
  constexpr int NW = kGatherThreads / 32;
  __shared__ float red_v[NW * BPW * TB];
  __shared__ int red_i[NW * BPW * TB];

  const int tb = blockIdx.x;
  int64_t entry0, nb;
  TileDesc td{};
  const int4* win;
  if (a.full) {
    entry0 = (int64_t)blockIdx.y * a.chunk_bins;
    nb = a.G - entry0 < a.chunk_bins ? a.G - entry0 : a.chunk_bins;
    win = a.win;
  } else {
    td = a.tiles[blockIdx.y];
    entry0 = td.entry_off;
    nb = (int64_t)td.wx * td.wy * td.wz;
    win = a.win + (int64_t)blockIdx.y * a.P;
  }

  // ---- stage the windows: rows (base + r) mod M of every pair
  constexpr int CPR = TB * (int)sizeof(E) / 16;  // 16-byte chunks per row
  const E* spec = static_cast<const E*>(a.spec) + (int64_t)tb * a.P * a.M * TB;
  for (int p = 0; p < a.P; ++p) {
    const int4 w = win[p];
    const uint4* src = reinterpret_cast<const uint4*>(spec + (int64_t)p * a.M * TB);
    uint4* dst = reinterpret_cast<uint4*>(sm + (int64_t)w.z * TB);
    const int n = w.y * CPR;
    for (int c = threadIdx.x; c < n; c += kGatherThreads) {
      const int r = c / CPR, q = c - r * CPR;
      int gi = w.x + r;
      while (gi >= a.M) gi -= a.M;
      dst[c] = __ldg(src + (int64_t)gi * CPR + q);
    }
  }
  __syncthreads();

  // ---- gather
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / TB, t = lane % TB;
  float best = -1.0f;
  int blb = -1;
  for (int64_t lb = warp * BPW + sub; lb < nb; lb += NW * BPW) {
    const uint16_t* rw = a.rows + (entry0 + lb) * a.p4;
    float acc = 0.0f;
    for (int p0 = 0; p0 < a.P; p0 += 4) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(rw + p0));
      const int rr[4] = {(int)(v.x & 0xffffu), (int)(v.x >> 16), (int)(v.y & 0xffffu),
                         (int)(v.y >> 16)};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (p0 + q >= a.P) break;
        if constexpr (!K3) {
          acc += sm[rr[q] * TB + t];
        } else {
          const float2* cf = a.coef3 + ((entry0 + lb) * a.P + p0 + q) * 3;
          const float2 c0 = __ldg(cf), c1 = __ldg(cf + 1), c2 = __ldg(cf + 2);
          const float2 z0 = sm[rr[q] * TB + t];
          const float2 z1 = sm[(rr[q] + 1) * TB + t];
          const float2 z2 = sm[(rr[q] + 2) * TB + t];
          const float vr = c0.x * z0.x - c0.y * z0.y + c1.x * z1.x - c1.y * z1.y +
                           c2.x * z2.x - c2.y * z2.y;
          const float vi = c0.x * z0.y + c0.y * z0.x + c1.x * z1.y + c1.y * z1.x +
                           c2.x * z2.y + c2.y * z2.x;
          const float pw = vr * vr + vi * vi;
          acc += MAG ? sqrtf(pw) : pw;
        }
      }
    }
    if constexpr (MAPMODE) {
      const int trial = tb * TB + t;
      if (trial < a.T) {
        int64_t gb = entry0 + lb;
        if (!a.full) {
          const int64_t lx = lb % td.wx, ly = (lb / td.wx) % td.wy,
                        lz = lb / ((int64_t)td.wx * td.wy);
          gb = (td.x0 + lx) + (int64_t)a.grid.n[0] * ((td.y0 + ly) + (int64_t)a.grid.n[1] * (td.z0 + lz));
        }
        a.map[(int64_t)trial * a.G + gb] = acc;
      }
    } else {
      if (acc > best) {
        best = acc;
        blb = (int)lb;
      }
    }
  }
  if constexpr (!MAPMODE) {
    red_v[(warp * BPW + sub) * TB + t] = best;
    red_i[(warp * BPW + sub) * TB + t] = blb;
    __syncthreads();
    if (threadIdx.x < TB) {
      float bv = -1.0f;
      int bi = -1;
      for (int s = 0; s < NW * BPW; ++s) {
        const float v = red_v[s * TB + threadIdx.x];
        const int i = red_i[s * TB + threadIdx.x];
        if (i < 0) continue;
        if (v > bv || (v == bv && i < bi)) {
          bv = v;
          bi = i;
        }
      }
      const int trial = tb * TB + threadIdx.x;
      if (trial < a.T && bi >= 0) {
        int64_t gb = entry0 + bi;
        if (!a.full) {
          const int64_t lx = bi % td.wx, ly = (bi / td.wx) % td.wy,
                        lz = bi / ((int64_t)td.wx * td.wy);
          gb = (td.x0 + lx) + (int64_t)a.grid.n[0] * ((td.y0 + ly) + (int64_t)a.grid.n[1] * (td.z0 + lz));
        }
        const unsigned long long key =
            ((unsigned long long)__float_as_uint(bv) << 32) | (0xffffffffull - (unsigned long long)gb);
        atomicMax(a.keys + trial, key);
      }
    }
  }
}

__global__ void k_decode_keys(const unsigned long long* keys, int T, int64_t* idx, float* val) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const unsigned long long k = keys[t];
  if (k == 0ull) {
    idx[t] = -1;
    val[t] = 0.0f;
    return;
  }
  idx[t] = (int64_t)(0xffffffffull - (k & 0xffffffffull));
  val[t] = __uint_as_float((unsigned)(k >> 32));
}

template <int TB, bool K3, bool MAG, bool MAPMODE>
void run(Ctx* ctx, const GatherArgs& a, dim3 grid, size_t smem) {
  auto kern = k_gather<TB, K3, MAG, MAPMODE>;
  GH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  KTimer kt(ctx, "gather");
  kern<<<grid, kGatherThreads, smem, ctx->stream>>>(a);
  GH_LAUNCHED(ctx);
}

template <int TB, bool K3>
void dispatch(Ctx* ctx, const GatherArgs& a, dim3 grid, size_t smem, bool mag, bool mapmode) {
  if (mapmode) {
    if (mag) run<TB, K3, true, true>(ctx, a, grid, smem);
    else run<TB, K3, false, true>(ctx, a, grid, smem);
  } else {
    if (mag) run<TB, K3, true, false>(ctx, a, grid, smem);
    else run<TB, K3, false, false>(ctx, a, grid, smem);
  }
}

}  // namespace

void launch_gather(Ctx* ctx, Table* t, const void* spec_d, int T, int combine, float* map_d,
                   unsigned long long* keys_d) {
  const Plan& pl = t->plan;
  GatherArgs a{};
  a.spec = spec_d;
  a.tiles = pl.tiles_d;
  a.win = pl.win_d;
  a.rows = pl.rows_d;
  a.coef3 = pl.coef3_d;
  a.grid = t->grid;
  a.G = t->G;
  a.full = pl.full;
  a.P = t->P;
  a.p4 = pl.p4;
  a.M = t->M;
  a.T = T;
  a.map = map_d;
  a.keys = keys_d;
  const int n_tb = (T + pl.tb - 1) / pl.tb;
  int n_cols = pl.n_tiles;
  if (pl.full) {
    // split the bins so that ~2 waves of CTAs exist, but keep >= 4096 bins
    // per CTA to amortise the staging of the whole ring
    int64_t chunks = (2LL * ctx->num_sms + n_tb - 1) / n_tb;
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, (t->G + 4095) / 4096));
    a.chunk_bins = (t->G + chunks - 1) / chunks;
    n_cols = static_cast<int>((t->G + a.chunk_bins - 1) / a.chunk_bins);
  }
  if (n_cols > 65535) fail(GH_EINVAL, "gather: too many location tiles for one launch");
  const size_t smem = static_cast<size_t>(pl.max_rows) * pl.tb * pl.esize;
  dim3 grid(n_tb, n_cols);
  const bool mag = combine == GH_MAGNITUDE;
  const bool mapmode = map_d != nullptr;
  if (!pl.k3) {
    // K = 1: the FFT epilogue already wrote power or magnitude
    if (pl.tb == 16) dispatch<16, false>(ctx, a, grid, smem, false, mapmode);
    else dispatch<32, false>(ctx, a, grid, smem, false, mapmode);
  } else {
    if (pl.tb != 16) fail(GH_EINVAL, "gather: complex plans use 16-trial batches");
    dispatch<16, true>(ctx, a, grid, smem, mag, mapmode);
  }
}

void launch_decode_keys(Ctx* ctx, const unsigned long long* keys_d, int T, int64_t* idx_d,
                        float* val_d) {
  KTimer kt(ctx, "decode");
  k_decode_keys<<<(T + 255) / 256, 256, 0, ctx->stream>>>(keys_d, T, idx_d, val_d);
  GH_LAUNCHED(ctx);
}

}  // namespace gh
