// gh_gather_common.cuh — pieces shared by the gather kernels (gh_gather_impl.cuh)
// and the fused top-K gather (gh_gather_topk.cu): the launch arguments and
// the per-pair accumulate step.
#pragma once
#include <cuda_runtime.h>

#include "gh_internal.cuh"
#include "gh_ptx.cuh"

namespace gh {
namespace {

struct GatherArgs {
  const void* spec;       // [batches][P][M][TB] float or float2
  const TileDesc* tiles;  // tiled plan
  const int4* win;        // [tiles][P] / [P]
  const uint16_t* rows;   // [p4 / 4][entries][4], 16-byte units (word-major)
  int64_t n_entries;      // entries of the plan (word stride of rows)
  const float2* coef3;    // [P][3][entries] (word-major), complex weights (poly3, linear)
  const float4* coefr;    // [P][entries] real weights (w0, w1, w2, 0): polar tables, else null
  const uint32_t* binid;  // [entries] global bin (bank-permuted full plan), or null
  int64_t tie_from;       // permuted plan: entries from here on are not in per-lane bin order
  const uint32_t* crow;   // [entries] compact rows: P ring rows of cbits each, or null
  int cbits;              // bits per ring row in crow
  int ring;               // staged rows per pair (full-ring plan)
  gh_grid grid;
  int64_t G;              // bins of the table (shard)
  int64_t bin0;           // global index of the shard's first bin
  int n_batches;          // trial batches (full plan: persistent work split)
  int batch_group;        // persistent tiled gather: batches per group (items group-major)
  int n_tiles;            // tiled plan
  int chunk_pairs;        // tiled plan: pairs per staging chunk
  int full;
  int P, p4, M, T;
  float* map;             // parity mode [T][G]
  unsigned long long* keys;
};

__device__ __forceinline__ float2 f2(float x, float y) { return make_float2(x, y); }

// value contribution of one pair for the lane's trials
template <int TB, bool K3, bool MAG, int L>
__device__ __forceinline__ void accumulate(const float4* __restrict__ smv, unsigned off16,
                                           const float2* __restrict__ cf, float2 (&acc)[2],
                                           bool first, int64_t cs = 0,
                                           const float4* __restrict__ cr = nullptr) {
  if constexpr (!K3) {
    const float4 z = smv[off16];
    if (first) {
      acc[0] = f2(z.x, z.y);
      acc[1] = f2(z.z, z.w);
    } else {
      acc[0] = __fadd2_rn(acc[0], f2(z.x, z.y));
      acc[1] = __fadd2_rn(acc[1], f2(z.z, z.w));
    }
  } else {
    const float4 z0 = smv[off16];
    const float4 z1 = smv[off16 + L];
    const float4 z2 = smv[off16 + 2 * L];
    float2 ra, rb;
    if (cr) {
      // real weights (polar interpolation): one 16-byte load, 3 FFMA2 per trial
      const float4 w = __ldg(cr);
      ra = __fmul2_rn(f2(w.x, w.x), f2(z0.x, z0.y));
      ra = __ffma2_rn(f2(w.y, w.y), f2(z1.x, z1.y), ra);
      ra = __ffma2_rn(f2(w.z, w.z), f2(z2.x, z2.y), ra);
      rb = __fmul2_rn(f2(w.x, w.x), f2(z0.z, z0.w));
      rb = __ffma2_rn(f2(w.y, w.y), f2(z1.z, z1.w), rb);
      rb = __ffma2_rn(f2(w.z, w.z), f2(z2.z, z2.w), rb);
    } else {
      const float2 c0 = __ldg(cf), c1 = __ldg(cf + cs), c2 = __ldg(cf + 2 * cs);
      // trial a = (x, y), trial b = (z, w); v = sum_j c_j z_j (complex product)
      ra = __fmul2_rn(f2(c0.x, c0.x), f2(z0.x, z0.y));           // (c0r*zr, c0r*zi)
      ra = __ffma2_rn(f2(-c0.y, c0.y), f2(z0.y, z0.x), ra);      // (-c0i*zi, c0i*zr)
      ra = __ffma2_rn(f2(c1.x, c1.x), f2(z1.x, z1.y), ra);
      ra = __ffma2_rn(f2(-c1.y, c1.y), f2(z1.y, z1.x), ra);
      ra = __ffma2_rn(f2(c2.x, c2.x), f2(z2.x, z2.y), ra);
      ra = __ffma2_rn(f2(-c2.y, c2.y), f2(z2.y, z2.x), ra);
      rb = __fmul2_rn(f2(c0.x, c0.x), f2(z0.z, z0.w));
      rb = __ffma2_rn(f2(-c0.y, c0.y), f2(z0.w, z0.z), rb);
      rb = __ffma2_rn(f2(c1.x, c1.x), f2(z1.z, z1.w), rb);
      rb = __ffma2_rn(f2(-c1.y, c1.y), f2(z1.w, z1.z), rb);
      rb = __ffma2_rn(f2(c2.x, c2.x), f2(z2.z, z2.w), rb);
      rb = __ffma2_rn(f2(-c2.y, c2.y), f2(z2.w, z2.z), rb);
    }
    const float2 sq = __ffma2_rn(f2(ra.x, rb.x), f2(ra.x, rb.x),
                                 __fmul2_rn(f2(ra.y, rb.y), f2(ra.y, rb.y)));
    const float2 v = MAG ? f2(sqrtf(sq.x), sqrtf(sq.y)) : sq;
    if (first) acc[0] = v;
    else acc[0] = __fadd2_rn(acc[0], v);
  }
}

// Persistent tiled gathers walk items group-major: groups of `batch_group`
// trial batches, and inside a group tile-major, so the plan rows of a tile
// are read once per group (its batches run together on neighbouring CTAs:
// L2 hits) while the group's spectra stay L2-resident. item -> (tile, batch).
__device__ __forceinline__ void item_tile_batch(const GatherArgs& a, int64_t item, int* tile,
                                                int* tb) {
  const int bg = a.batch_group;
  const int full = a.n_batches / bg;
  const int64_t per_group = (int64_t)a.n_tiles * bg;
  if (item < full * per_group) {
    const int g = (int)(item / per_group);
    const int r = (int)(item - g * per_group);
    *tile = r / bg;
    *tb = g * bg + r % bg;
  } else {
    const int bl = a.n_batches - full * bg;  // last, partial group
    const int r = (int)(item - full * per_group);
    *tile = r / bl;
    *tb = full * bg + r % bl;
  }
}

}  // namespace
}  // namespace gh
