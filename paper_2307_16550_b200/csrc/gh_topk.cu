// gh_topk.cu — per-trial top-K local maxima of a decision map (sm_100a).
//
// BASELINE c3 (K = 5 targets, "top-5 local-maximum peak pick"): a bin is a
// local maximum if its value is > every lattice neighbour with a smaller
// index and >= every neighbour with a larger index (8 neighbours in 2-D, 26
// in 3-D; plateaus resolve to their smallest index, the argmax_index tie
// rule of src/direct.cpp:55-62). Candidates rank by (value desc, index asc).
// Restates oracle/gridhop_oracle.cpp or_topk_local_max.
//
// One CTA per trial streams the map once with float4 loads (four in flight
// per thread). Ranking uses the 64-bit key (orderable value bits << 32 |
// 2^32-1-index), so "better" is one unsigned compare. Each warp keeps a
// sorted top-K list in lanes 0..K-1 and a prune key: the K-th key of any
// verified list in the CTA (a value below it has K verified local maxima
// above it, so pruning is exact). Per step the warp ballots the lanes whose
// element beats the prune key — rare once the lists fill — and queues them
// in shared memory; 32 queued candidates are tested in one parallel round
// (lane l tests candidate l, its neighbour loads issued together) and the
// local maxima enter the list by shuffle inserts. No lane waits alone on
// dependent neighbour loads, which is what made a per-thread version
// divergence-bound.
#include <cuda_runtime.h>

#include "gh_internal.cuh"

namespace gh {
namespace {

constexpr int kTopkThreads = 512;
constexpr int kMaxK = 8;
constexpr int kVec = 4;  // float4 loads in flight per thread and iteration
constexpr int kQueue = 160;

// order-preserving float -> uint32 (larger float -> larger uint)
__device__ __forceinline__ uint32_t ord(float v) {
  const uint32_t b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
__device__ __forceinline__ unsigned long long mkkey(float v, uint32_t i) {
  return ((unsigned long long)ord(v) << 32) | (0xffffffffu - i);
}

struct WarpTopK {
  unsigned long long e;    // lane k < cnt: k-th best key of this warp (sorted desc)
  int cnt;                 // valid entries (warp-uniform)
  unsigned long long thr;  // prune key (warp-uniform): skip keys <= thr
  int qn;                  // queued candidates (warp-uniform)
};

// local-maximum test of one candidate key (per lane; neighbours loaded
// together so one lane pays one memory latency)
__device__ __forceinline__ bool is_local_max(const float* __restrict__ m, unsigned long long ck,
                                             int nx, int ny, int nz) {
  const uint32_t ci = 0xffffffffu - static_cast<uint32_t>(ck);
  const float cv = unord(static_cast<uint32_t>(ck >> 32));
  const uint32_t nxy = (uint32_t)nx * (uint32_t)ny;
  const int x = (int)(ci % (uint32_t)nx), y = (int)((ci / (uint32_t)nx) % (uint32_t)ny);
  const int z = (int)(ci / nxy);
  bool ok = true;
  for (int dz = (nz > 1 ? -1 : 0); dz <= (nz > 1 ? 1 : 0); ++dz) {
    const int zz = z + dz;
    if (zz < 0 || zz >= nz) continue;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const int yy = y + dy;
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int xx = x + dx;
        if ((dx == 0 && dy == 0 && dz == 0) || yy < 0 || yy >= ny || xx < 0 || xx >= nx) continue;
        const uint32_t j = ((uint32_t)zz * (uint32_t)ny + (uint32_t)yy) * (uint32_t)nx + (uint32_t)xx;
        const float nv = __ldg(m + j);
        ok &= (j < ci) ? (cv > nv) : (cv >= nv);
      }
    }
  }
  return ok;
}

// Test the queued candidates (lane l takes candidate l) and insert the local
// maxima into the warp list. All lanes must call.
__device__ __forceinline__ void warp_flush(WarpTopK& w, unsigned long long* q,
                                           const float* __restrict__ m, int K, int nx, int ny,
                                           int nz, unsigned long long* cta_thr) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  const int n = w.qn < 32 ? w.qn : 32;
  const unsigned long long ck = lane < n ? q[lane] : 0ull;
  const bool cand = lane < n && ck > w.thr;
  unsigned ok = __ballot_sync(0xffffffffu, cand && is_local_max(m, ck, nx, ny, nz));
  // keep the overflow (at most 31) queued
  const int rest = w.qn - n;
  for (int b = 0; b < rest; b += 32) {  // shift the overflow down by 32
    const unsigned long long moved = b + lane < rest ? q[32 + b + lane] : 0ull;
    __syncwarp();
    if (b + lane < rest) q[b + lane] = moved;
    __syncwarp();
  }
  w.qn = rest;
  while (ok) {
    const int src = __ffs(ok) - 1;
    ok &= ok - 1;
    const unsigned long long c = __shfl_sync(0xffffffffu, ck, src);
    if (c <= w.thr) continue;
    const int pos = __popc(__ballot_sync(0xffffffffu, lane < w.cnt && w.e > c));
    const unsigned long long up = __shfl_up_sync(0xffffffffu, w.e, 1);
    if (lane > pos) w.e = up;
    if (lane == pos) w.e = c;
    if (w.cnt < K) ++w.cnt;
    if (w.cnt == K) {
      const unsigned long long kth = __shfl_sync(0xffffffffu, w.e, K - 1);
      if (kth > w.thr) {
        w.thr = kth;
        if (lane == 0) atomicMax(cta_thr, kth);
      }
    }
  }
}

// Offer one element per lane (act = lane has one): elements above the prune
// key are queued; a full queue (>= 32) is tested in one parallel round. All
// lanes must call.
__device__ __forceinline__ void warp_offer(WarpTopK& w, unsigned long long* q,
                                           const float* __restrict__ m, float v, uint32_t i,
                                           bool act, int K, int nx, int ny, int nz,
                                           unsigned long long* cta_thr) {
  const int lane = threadIdx.x & 31;
  const unsigned long long key = act ? mkkey(v, i) : 0ull;
  const unsigned pend = __ballot_sync(0xffffffffu, key > w.thr);
  if (!pend) return;
  if (key > w.thr) q[w.qn + __popc(pend & ((1u << lane) - 1u))] = key;
  w.qn += __popc(pend);
}

// Candidates are the elements [e0, e1) of each trial's map (a shard's core
// layers); neighbours are read over the whole map (its halo layers too).
__global__ void __launch_bounds__(kTopkThreads) k_topk_localmax(const float* __restrict__ map,
                                                               int64_t G, int nx, int ny, int nz,
                                                               int K, int64_t bin0, int64_t e0,
                                                               int64_t e1, int64_t* idx_out,
                                                               float* val_out) {
  constexpr int NW = kTopkThreads / 32;
  __shared__ unsigned long long cta_thr;
  __shared__ unsigned long long lists[NW][kMaxK];
  __shared__ int counts[NW];
  // per-warp candidates awaiting the test: up to 31 + 4 offers of 32 between
  // flushes (one flush site per float4 keeps the unrolled loop small enough
  // for the instruction cache)
  __shared__ unsigned long long queue[NW][kQueue];
  const int trial = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* m = map + (int64_t)trial * G;
  const float* mc = m + e0;  // the scanned range
  const int64_t Gc = e1 - e0;
  if (threadIdx.x == 0) cta_thr = 0ull;
  __syncthreads();
  WarpTopK w{0ull, 0, 0ull, 0};
  unsigned long long* wq = queue[warp];
  // scalar head up to 16-byte alignment, float4 body, scalar tail; loops
  // have warp-uniform trip counts (inactive lanes offer nothing)
  const int64_t lead = (int64_t)((16 - (reinterpret_cast<uintptr_t>(mc) & 15)) & 15) / 4;
  const int64_t h = lead < Gc ? lead : Gc;
  for (int64_t b = 0; b < h; b += kTopkThreads) {
    const int64_t i = b + threadIdx.x;
    const bool act = i < h;
    warp_offer(w, wq, m, act ? __ldg(mc + i) : 0.f, (uint32_t)(e0 + i), act, K, nx, ny, nz,
               &cta_thr);
    while (w.qn >= 32) warp_flush(w, wq, m, K, nx, ny, nz, &cta_thr);
  }
  const float4* m4 = reinterpret_cast<const float4*>(mc + h);
  const int64_t n4 = (Gc - h) / 4;
  for (int64_t g0 = 0; g0 < n4; g0 += (int64_t)kTopkThreads * kVec) {
    float4 q[kVec];
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      const int64_t g = g0 + (int64_t)u * kTopkThreads + threadIdx.x;
      q[u] = g < n4 ? __ldg(m4 + g) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const unsigned long long ct = *reinterpret_cast<volatile unsigned long long*>(&cta_thr);
    if (ct > w.thr) w.thr = ct;
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      const int64_t g = g0 + (int64_t)u * kTopkThreads + threadIdx.x;
      const bool act = g < n4;
      const uint32_t i = (uint32_t)(e0 + h + 4 * g);
      // float pre-filter: key > prune key implies value >= its value, so a
      // float4 whose four values are all below it is skipped in one vote
      const float tv = w.thr ? unord(static_cast<uint32_t>(w.thr >> 32)) : -INFINITY;
      const bool any4 = act && (q[u].x >= tv || q[u].y >= tv || q[u].z >= tv || q[u].w >= tv);
      if (!__any_sync(0xffffffffu, any4)) continue;
      warp_offer(w, wq, m, q[u].x, i, act, K, nx, ny, nz, &cta_thr);
      warp_offer(w, wq, m, q[u].y, i + 1, act, K, nx, ny, nz, &cta_thr);
      warp_offer(w, wq, m, q[u].z, i + 2, act, K, nx, ny, nz, &cta_thr);
      warp_offer(w, wq, m, q[u].w, i + 3, act, K, nx, ny, nz, &cta_thr);
      while (w.qn >= 32) warp_flush(w, wq, m, K, nx, ny, nz, &cta_thr);
    }
  }
  for (int64_t b = h + 4 * n4; b < Gc; b += kTopkThreads) {
    const int64_t i = b + threadIdx.x;
    const bool act = i < Gc;
    warp_offer(w, wq, m, act ? __ldg(mc + i) : 0.f, (uint32_t)(e0 + i), act, K, nx, ny, nz,
               &cta_thr);
    while (w.qn >= 32) warp_flush(w, wq, m, K, nx, ny, nz, &cta_thr);
  }
  while (w.qn > 0) warp_flush(w, wq, m, K, nx, ny, nz, &cta_thr);
  if (lane < K) lists[warp][lane] = lane < w.cnt ? w.e : 0ull;
  if (lane == 0) counts[warp] = w.cnt;
  __syncthreads();
  // merge the NW warp lists: K rounds of "largest remaining key"; lane l
  // walks warp l's list
  if (warp == 0) {
    int head = 0;
    for (int k = 0; k < K; ++k) {
      const unsigned long long mine =
          (lane < NW && head < counts[lane]) ? lists[lane][head] : 0ull;
      unsigned long long best = mine;
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other > best ? other : best;
      }
      if (best != 0ull && mine == best) ++head;  // keys are unique: one owner
      if (lane == 0) {
        const bool valid = best != 0ull;
        idx_out[(int64_t)trial * K + k] =
            valid ? bin0 + (int64_t)(0xffffffffu - static_cast<uint32_t>(best)) : -1;
        val_out[(int64_t)trial * K + k] = valid ? unord(static_cast<uint32_t>(best >> 32)) : 0.0f;
      }
    }
  }
}

}  // namespace

void launch_topk(Ctx* ctx, const float* map_d, int T, const gh_grid& g, int K, int64_t bin0,
                 int64_t* idx_d, float* val_d, int64_t e0, int64_t e1) {
  if (K < 1 || K > kMaxK) fail(GH_EINVAL, "top-k: k must be in [1, 8]");
  const int64_t G = (int64_t)g.n[0] * g.n[1] * g.n[2];
  if (G >= 0xffffffffll) fail(GH_EINVAL, "top-k: map above 2^32 - 1 bins");
  if (e1 < 0) e1 = G;
  if (e0 < 0 || e0 >= e1 || e1 > G) fail(GH_EINVAL, "top-k: core range outside the map");
  KTimer kt(ctx, "topk");
  k_topk_localmax<<<T, kTopkThreads, 0, ctx->stream>>>(map_d, G, g.n[0], g.n[1], g.n[2], K, bin0,
                                                       e0, e1, idx_d, val_d);
  GH_LAUNCHED(ctx);
}

}  // namespace gh
