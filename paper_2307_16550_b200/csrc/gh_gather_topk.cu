// gh_gather_topk.cu — BASELINE c3's fused gather + top-K local-maximum
// pick (sm_100a). The gather is the one of gh_gather_impl.cuh (hopping.cpp:59-117
// hop_bin_value with Mc = 1); the pick is the rule of or_topk_local_max /
// k_topk_localmax (ties to the smallest bin, direct.cpp:55-62).
#include <cuda_runtime.h>

#include <algorithm>

#include "gh_gather_common.cuh"

#ifdef GH_TOPK_PROF
// diagnostic build (tools/topk_prof.sh): per-phase SM cycles summed over warps
__device__ unsigned long long g_topk_prof[16];
#define PROF_COUNT(i) atomicAdd(&g_topk_prof[i], 1ull)
#define PROF_MARK(i)                                                                        \
  do {                                                                                      \
    const long long _t = clock64();                                                         \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_topk_prof[i], (unsigned long long)(_t - _pt)); \
    _pt = _t;                                                                               \
  } while (0)
#else
#define PROF_MARK(i) \
  do {               \
  } while (0)
#define PROF_COUNT(i) \
  do {                \
  } while (0)
#endif

namespace gh {
namespace {

using namespace ptx;

// ---- fused top-K (BASELINE c3): gather + local-maximum pick per tile.
//
// Halo plans (build_plan_topk): a tile's box is its core grown by one bin,
// so the gather computes every value a core bin's local-maximum test reads.
// Values live in shared memory, one plane per trial, box (x, y) at
// (y + 1) * pitch + x + 1: a one-cell ring around the box holds -inf, so the
// neighbours of a core bin on a grid edge read -inf (no bounds tests).
//
// Persistent CTAs (one per SM) walk (tile, batch) items batch-major with
// two warp roles, so the pick of item i runs while item i + 1 is gathered:
//  * NG gather warps: wait until the values planes of buffer i % 2 are free,
//    write their -inf ring, gather as k_gather (8-trial power rows, LDS.128
//    per pair, FADD2) into them, and keep per trial the largest core value of
//    their band of the box. A named barrier among them marks the windows
//    dead: one gather warp issues the next item's window staging (TMA bulk
//    copies, one pair per lane), then all signal the planes ready.
//  * NP pick warps, one trial each: the prune key (value bits << 32 | ~bin)
//    is the larger of the trial's global key (the K-th key of a finished
//    tile) and the K-th best band maximum that passes the local-maximum test
//    (> smaller-index neighbours, >= larger ones: the rule of
//    k_topk_localmax / or_topk_local_max). Either is the K-th key of K
//    distinct maxima, so it bounds the trial's K-th maximum from below and
//    pruning is exact. The warp filters the trial's core rows 4 values per
//    LDS.128 (half a warp per row); values at or above the prune value get
//    the full test, maxima above the key enter the warp's candidate list;
//    its K best -> cand[trial][tile][K], the global key is raised, the
//    planes are released. A list that overflows is replaced by an exact row
//    scan of the core by that warp.
// Buffers hand over through named barriers (ready: gather warps arrive, pick
// warps wait; free: the reverse). Maps never reach HBM (c3: 4 MB per trial).
constexpr int kTopkNG = 16;  // gather warps
constexpr int kTopkNP = 8;   // pick warps (one per trial of the 8-trial batch)
constexpr int kTopkNW = kTopkNG + kTopkNP;
constexpr int kTopkMaxK = 8;
constexpr int kTopkCap = 64;    // candidate keys per trial and item
constexpr int kTopkStrip = 30;  // fallback row scan: core x per lane strip (lanes 1..30)
constexpr int kBarGather = 1, kBarReady = 2, kBarFree = 4;  // named barrier ids (+ buffer)

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct TopkArgs {
  int K;
  unsigned long long* cand;  // [T][n_tiles][K] keys, 0 = none
  unsigned long long* thr;   // [T] prune keys (K-th key of a finished tile)
  unsigned vals_off;         // byte offset of the values planes in dynamic shared memory
  int plane;                 // floats per trial plane
  const uint16_t* pos;       // [entries] plane position | 0x8000 for halo bins (plan pos_d)
};

__device__ __forceinline__ uint32_t ord_f(float v) {
  const uint32_t b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ float key_value(unsigned long long k) {  // non-negative values
  return __uint_as_float((uint32_t)(k >> 32) & 0x7fffffffu);
}

// local maximum at plane position q (ring layout: every neighbour readable):
// strictly above the smaller-index neighbours, at least the larger ones
__device__ __forceinline__ bool is_lm(const float* pl, int q, int pitch, float c) {
  const float s = fmaxf(fmaxf(pl[q - pitch - 1], pl[q - pitch]), fmaxf(pl[q - pitch + 1], pl[q - 1]));
  const float w = fmaxf(fmaxf(pl[q + pitch - 1], pl[q + pitch]), fmaxf(pl[q + pitch + 1], pl[q + 1]));
  return c > s && c >= w;
}

// insert key ck into the warp's sorted register list (lane k < K: k-th key)
__device__ __forceinline__ void list_insert(unsigned long long& mine, unsigned long long ck, int K,
                                            int lane) {
  const int pos = __popc(__ballot_sync(0xffffffffu, lane < K && mine > ck));
  const unsigned long long up = __shfl_up_sync(0xffffffffu, mine, 1);
  if (lane < K && lane > pos) mine = up;
  if (lane == pos) mine = ck;  // pos < K: ck beats the K-th (or a free slot)
}

template <int PC, int PQ>
__global__ void __launch_bounds__(kTopkNW * 32, 1) k_gather_topk(GatherArgs a, TopkArgs tk) {
  constexpr int TB = 8, L = 2, BPW = 16, NG = kTopkNG, NP = kTopkNP;
  constexpr int SW = NG - 1;  // the gather warp that issues the staging
  static_assert(NP == TB, "one pick warp per trial");
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t stage_bar;
  __shared__ unsigned long long cbuf[TB][kTopkCap];
  __shared__ float regv[2][TB][NG];  // band maxima per buffer
  __shared__ int regp[2][TB][NG];    // ... and their plane positions
  const int P = PC ? PC : a.P;
  const int K = tk.K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n_items = (int64_t)a.n_tiles * a.n_batches;
  if ((int64_t)blockIdx.x >= n_items) return;
  const int nx = a.grid.n[0];

  // the item's windows by TMA bulk copies, one pair per lane of warp SW (the
  // window descriptors load in parallel)
  auto stage = [&](int64_t item) {
    const int tile = (int)(item % a.n_tiles), tb = (int)(item / a.n_tiles);
    const int4* win = a.win + (int64_t)tile * a.P;
    const uint4* spec = reinterpret_cast<const uint4*>(static_cast<const unsigned char*>(a.spec) +
                                                       (int64_t)tb * a.P * a.M * TB * 4);
    uint4* sm4 = reinterpret_cast<uint4*>(smraw);
    uint32_t total = 0;
    for (int p = lane; p < P; p += 32) total += (uint32_t)__ldg(&win[p].y) * 16u * L;
    for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
    if (lane == 0) mbar_expect_tx(&stage_bar, total);
    __syncwarp();
    for (int p = lane; p < P; p += 32) {
      const int4 w = __ldg(&win[p]);
      const uint4* src = spec + (int64_t)p * a.M * L;
      uint4* dst = sm4 + (int64_t)w.z * L;
      for (int r = 0, gi = w.x; r < w.y; gi = 0) {
        const int n = a.M - gi < w.y - r ? a.M - gi : w.y - r;
        bulk_g2s(dst + (int64_t)r * L, src + (int64_t)gi * L, (uint32_t)n * 16u * L, &stage_bar);
        r += n;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&stage_bar);
  };

  if (threadIdx.x == SW * 32) {
    mbar_init(&stage_bar, 1);
    mbar_fence_init();
  }
  __syncwarp();
  if (warp == SW) stage(blockIdx.x);
  __syncthreads();  // barrier initialised

  if (warp < NG) {
    // ================= gather warps
#ifdef GH_TOPK_PROF
    long long _pt = clock64();
#endif
    uint32_t phase = 0;
    const int sub = lane / L, v = lane % L;
    const float4* smv = reinterpret_cast<const float4*>(smraw) + v;
    const int pq = PC ? (PC + 3) / 4 : (a.p4 >> 2);
    const uint2* rows2 = reinterpret_cast<const uint2*>(a.rows);
    int it = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const int b = it & 1;
      const int tile = (int)(item % a.n_tiles);
      const TileDesc td = a.tiles[tile];
      const int64_t entry0 = td.entry_off;
      const int nb = td.wx * td.wy * td.wz;
      const int pitch = topk_pitch(td.wx);
      float* vals = reinterpret_cast<float*>(smraw + tk.vals_off) + (size_t)b * TB * tk.plane;
      if (it >= 2) named_sync(kBarFree + b, kTopkNW * 32);  // item it - 2 picked
      PROF_MARK(3);
      {  // -inf ring around the box (rows -1 and wy, columns -1 and wx)
        const int rw = td.wx + 2, nring = 2 * rw + 2 * td.wy;
        for (int i = threadIdx.x; i < TB * nring; i += NG * 32) {
          const int t = i / nring, r = i % nring;
          int q;
          if (r < rw) q = r;
          else if (r < 2 * rw) q = (td.wy + 1) * pitch + (r - rw);
          else if (r < 2 * rw + td.wy) q = (r - 2 * rw + 1) * pitch;
          else q = (r - 2 * rw - td.wy + 1) * pitch + td.wx + 1;
          vals[t * tk.plane + q] = -INFINITY;
        }
      }
      float rbest[4] = {-1.0f, -1.0f, -1.0f, -1.0f};  // this lane's largest core value per trial
      int rpos[4] = {-1, -1, -1, -1};                 // ... and its plane position
      const int per_warp = ((nb + NG - 1) / NG + BPW - 1) / BPW * BPW;
      const int w0 = warp * per_warp < nb ? warp * per_warp : nb;
      const int w1 = w0 + per_warp < nb ? w0 + per_warp : nb;
      uint2 cur[PQ], nxt[PQ];
#pragma unroll
      for (int q = 0; q < PQ; ++q) cur[q] = nxt[q] = make_uint2(0u, 0u);
      if (w0 + lane < w1) {
#pragma unroll
        for (int q = 0; q < PQ; ++q)
          if (q < pq) cur[q] = __ldg(rows2 + q * a.n_entries + entry0 + w0 + lane);
      }
      mbar_wait(&stage_bar, phase);
      PROF_MARK(0);
      phase ^= 1u;
      float* vout = vals + v * 4 * tk.plane;  // this lane's 4 trial planes
      for (int blk = w0; blk < w1; blk += 32) {
        if (blk + 32 + lane < w1) {
#pragma unroll
          for (int q = 0; q < PQ; ++q)
            if (q < pq) nxt[q] = __ldg(rows2 + q * a.n_entries + entry0 + blk + 32 + lane);
        }
        const int nblk = w1 - blk < 32 ? w1 - blk : 32;
        auto step = [&](int s, bool check) {
          const int j = s * BPW + sub;
          const int lb = blk + (!check || j < nblk ? j : 0);
          float2 acc[2];
          acc[0] = acc[1] = f2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < PQ; ++q) {
            if (q >= pq) break;
            const unsigned ex = __shfl_sync(0xffffffffu, cur[q].x, j & 31);
            const unsigned ey = __shfl_sync(0xffffffffu, cur[q].y, j & 31);
            const unsigned o[4] = {ex & 0xffffu, ex >> 16, ey & 0xffffu, ey >> 16};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int p = 4 * q + u;
              if (PC ? p >= PC : p >= a.P) break;
              accumulate<TB, false, false, L>(smv, o[u], nullptr, acc, p == 0);
            }
          }
          if (!check || j < nblk) {
            const int pe = __ldg(tk.pos + entry0 + lb);
            const int pos = pe & 0x7fff;
            const float vv[4] = {acc[0].x, acc[0].y, acc[1].x, acc[1].y};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              vout[i * tk.plane + pos] = vv[i];
              if (pe < 0x8000 && vv[i] > rbest[i]) {
                rbest[i] = vv[i];
                rpos[i] = pos;
              }
            }
          }
        };
        if (nblk == 32) {
#pragma unroll
          for (int s = 0; s < 32 / BPW; ++s) step(s, false);
        } else {
          for (int s = 0; s * BPW < nblk; ++s) step(s, true);
        }
#pragma unroll
        for (int q = 0; q < PQ; ++q) cur[q] = nxt[q];
      }
      // the warp's band maximum per trial (lanes 0 / 1 hold trials 0-3 / 4-7)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        for (int o = L; o < 32; o <<= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, rbest[i], o);
          const int op = __shfl_xor_sync(0xffffffffu, rpos[i], o);
          if (ov > rbest[i]) {
            rbest[i] = ov;
            rpos[i] = op;
          }
        }
        if (lane < L) {
          regv[b][v * 4 + i][warp] = rbest[i];
          regp[b][v * 4 + i][warp] = rpos[i];
        }
      }
      PROF_MARK(1);
      named_sync(kBarGather, NG * 32);  // windows no longer read
      PROF_MARK(2);
      if (warp == SW && item + gridDim.x < n_items) stage(item + gridDim.x);
      named_arrive(kBarReady + b, kTopkNW * 32);  // planes + band maxima of buffer b ready
    }
    // take the pick warps' last releases (every arrival has its wait)
    for (int k = it - 2 < 0 ? 0 : it - 2; k < it; ++k) named_sync(kBarFree + (k & 1), kTopkNW * 32);
    return;
  }

  // ================= pick warps: warp NG + t owns trial t of every batch
#ifdef GH_TOPK_PROF
  long long _pt = clock64();
#endif
  const int t = warp - NG;
  unsigned long long* cb = cbuf[t];
  int it = 0;
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
    const int b = it & 1;
    const int tile = (int)(item % a.n_tiles), tb = (int)(item / a.n_tiles);
    const int trial = tb * TB + t;
    // the global prune key: load it early (L2 latency under the wait)
    const unsigned long long g =
        trial < a.T ? *reinterpret_cast<volatile unsigned long long*>(tk.thr + trial) : 0ull;
    const TileDesc td = a.tiles[tile];
    const int pitch = topk_pitch(td.wx);
    const float* pl = reinterpret_cast<const float*>(smraw + tk.vals_off) +
                      ((size_t)b * TB + t) * tk.plane;
    named_sync(kBarReady + b, kTopkNW * 32);
    PROF_MARK(4);
    if (trial < a.T) {
      // prune key: the K-th best band maximum that is a local maximum
      // (distinct bands, distinct maxima), or the trial's global key
      float bv = -1.0f;
      if (lane < NG) {
        const int q = regp[b][t][lane];
        const float c = regv[b][t][lane];
        if (q >= 0 && is_lm(pl, q, pitch, c)) bv = c;
      }
      float kv = -1.0f;  // K-th best verified value; its smallest key bounds below
      for (int k = 0; k < K; ++k) {
        float m = bv;
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const unsigned own = __ballot_sync(0xffffffffu, bv == m);
        if (lane == __ffs(own) - 1) bv = -2.0f;
        kv = m;
      }
      const unsigned long long kth = kv >= 0.0f ? (unsigned long long)ord_f(kv) << 32 : 0ull;
      const unsigned long long thr = kth > g ? kth : g;
      const float tv = thr ? key_value(thr) : -1.0f;
      // filter: half a warp per core row, 4 plane values per LDS.128
      const int c0 = (td.cx0 + 1) >> 2, c1 = (td.cx0 + td.cwx + 1 + 3) >> 2;  // float4 columns
      const int nch = c1 - c0;
      int n = 0;  // candidates (warp-uniform)
      for (int y0 = td.cy0; y0 < td.cy0 + td.cwy; y0 += 2) {  // warp-uniform trips
        const int y = y0 + (lane >> 4);
        const bool yin = y < td.cy0 + td.cwy;
        const float* rp = pl + (y + 1) * pitch + 4 * c0;
        for (int cc0 = 0; cc0 < nch; cc0 += 16) {
          const int cc = cc0 + (lane & 15);
          float4 f = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
          if (cc < nch && yin) f = *reinterpret_cast<const float4*>(rp + 4 * cc);
          const bool any = fmaxf(fmaxf(f.x, f.y), fmaxf(f.z, f.w)) >= tv;
          if (!__any_sync(0xffffffffu, any)) continue;
          PROF_COUNT(8);
          const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int bx = 4 * (c0 + cc) + e - 1;  // box column
            unsigned long long key = 0ull;
            if (any && fv[e] >= tv && bx >= td.cx0 && bx < td.cx0 + td.cwx &&
                is_lm(pl, (y + 1) * pitch + bx + 1, pitch, fv[e])) {
              const int64_t gb = (int64_t)nx * (td.y0 + y) + td.x0 + bx;
              key = ((unsigned long long)ord_f(fv[e]) << 32) | (0xffffffffull - (uint64_t)gb);
              if (key < thr) key = 0ull;
            }
            const unsigned has = __ballot_sync(0xffffffffu, key != 0ull);
            if (key) {
              const int slot = n + __popc(has & ((1u << lane) - 1u));
              if (slot < kTopkCap) cb[slot] = key;
            }
            n += __popc(has);
          }
        }
      }
      __syncwarp();
      unsigned long long mine = 0ull;  // lane k < K: the k-th best key
      if (n <= kTopkCap) {
        unsigned long long x0 = lane < n ? cb[lane] : 0ull;
        unsigned long long x1 = lane + 32 < n ? cb[lane + 32] : 0ull;
        for (int k = 0; k < K; ++k) {
          const unsigned long long m = x0 > x1 ? x0 : x1;
          unsigned long long best = m;
          for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
            best = ob > best ? ob : best;
          }
          if (x0 == best) x0 = 0ull;
          else if (x1 == best) x1 = 0ull;
          if (lane == k) mine = best;
        }
      } else {
        PROF_COUNT(11);
        // list overflow: exact row scan of the whole core above the key
        unsigned long long sthr = thr;
        for (int strip = 0; strip * kTopkStrip < td.cwx; ++strip) {
          const int x = td.cx0 + strip * kTopkStrip - 1 + lane;  // box column of this lane
          const bool xin = x >= -1 && x <= td.wx;
          const bool centre = lane >= 1 && lane <= kTopkStrip && x < td.cx0 + td.cwx;
          const float* col = pl + x + 1;
          auto row = [&](int y, float& c, float& l, float& r, float& h) {
            c = xin ? col[(y + 1) * pitch] : -INFINITY;
            l = __shfl_up_sync(0xffffffffu, c, 1);
            r = __shfl_down_sync(0xffffffffu, c, 1);
            h = fmaxf(fmaxf(l, r), c);
          };
          float pc, pl_, pr, ph, x0, l0, r0, h0;
          row(td.cy0 - 1, pc, pl_, pr, ph);
          row(td.cy0, x0, l0, r0, h0);
          for (int y = td.cy0; y < td.cy0 + td.cwy; ++y) {
            float x1, l1, r1, h1;
            row(y + 1, x1, l1, r1, h1);
            const bool lm = centre && x0 > fmaxf(ph, l0) && x0 >= fmaxf(r0, h1);
            const int64_t gb = (int64_t)nx * (td.y0 + y) + td.x0 + x;
            const unsigned long long key =
                lm ? ((unsigned long long)ord_f(x0) << 32) | (0xffffffffull - (uint64_t)gb) : 0ull;
            unsigned ver = __ballot_sync(0xffffffffu, key != 0ull && key >= sthr);
            while (ver) {
              const int src = __ffs(ver) - 1;
              ver &= ver - 1;
              const unsigned long long ck = __shfl_sync(0xffffffffu, key, src);
              if (ck < sthr) continue;  // warp-uniform
              list_insert(mine, ck, K, lane);
              const unsigned long long k5 = __shfl_sync(0xffffffffu, mine, K - 1);
              sthr = k5 > sthr ? k5 : sthr;
            }
            ph = h0;
            x0 = x1;
            l0 = l1;
            r0 = r1;
            h0 = h1;
          }
        }
      }
      if (lane < K) tk.cand[((int64_t)trial * a.n_tiles + tile) * K + lane] = mine;
      const unsigned long long k5 = __shfl_sync(0xffffffffu, mine, K - 1);
      if (lane == 0 && k5) atomicMax(tk.thr + trial, k5);
    }
    PROF_MARK(5);
    named_arrive(kBarFree + b, kTopkNW * 32);  // buffer b free for item it + 2
  }
}

// Per trial: the K best of its tiles' candidate keys (keys are unique per
// bin, so the order is total), decoded to (bin, value); -1 = no maximum.
__global__ void k_topk_merge(const unsigned long long* __restrict__ cand, int T, int n_lists,
                             int K, int64_t* idx, float* val) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= T) return;
  const unsigned long long* c = cand + (int64_t)warp * n_lists;
  unsigned long long top[kTopkMaxK];
#pragma unroll
  for (int k = 0; k < kTopkMaxK; ++k) top[k] = 0ull;
  for (int i = lane; i < n_lists; i += 32) {  // per-lane sorted top-K
    unsigned long long x = __ldg(c + i);
#pragma unroll
    for (int k = 0; k < kTopkMaxK; ++k) {
      if (k < K && x > top[k]) {
        const unsigned long long y = top[k];
        top[k] = x;
        x = y;
      }
    }
  }
  int head = 0;
  for (int k = 0; k < K; ++k) {
    unsigned long long mine = 0ull;
#pragma unroll
    for (int j = 0; j < kTopkMaxK; ++j)
      if (j == head) mine = top[j];
    unsigned long long best = mine;
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other > best ? other : best;
    }
    if (best != 0ull && mine == best) ++head;
    if (lane == 0) {
      const bool ok = best != 0ull;
      idx[(int64_t)warp * K + k] = ok ? (int64_t)(0xffffffffull - (best & 0xffffffffull)) : -1;
      const uint32_t u = (uint32_t)(best >> 32);
      val[(int64_t)warp * K + k] = ok ? __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u)
                                      : 0.0f;
    }
  }
}

}  // namespace

void launch_gather_topk(Ctx* ctx, Table* t, const void* spec_d, int T, int K,
                        unsigned long long* cand_d, unsigned long long* thr_d) {
  const Plan& pl = t->plan_topk;
  if (!pl.built) fail(GH_ERUNTIME, "gather: top-K plan not built");
  if (K < 1 || K > kTopkMaxK) fail(GH_EINVAL, "top-k: k must be in [1, 8]");
  GatherArgs a{};
  a.spec = spec_d;
  a.tiles = pl.tiles_d;
  a.win = pl.win_d;
  a.rows = pl.rows_d;
  a.n_entries = pl.n_entries;
  a.grid = t->grid;
  a.G = t->G;
  a.P = t->P;
  a.p4 = pl.p4;
  a.M = t->M;
  a.T = T;
  a.n_batches = (T + pl.tb - 1) / pl.tb;
  a.n_tiles = pl.n_tiles;
  TopkArgs tk{};
  tk.K = K;
  tk.cand = cand_d;
  tk.thr = thr_d;
  const size_t win_bytes = ((size_t)pl.max_rows * pl.tb * pl.esize + 127) / 128 * 128;
  tk.vals_off = static_cast<unsigned>(win_bytes);
  tk.plane = pl.topk_plane;
  tk.pos = pl.pos_d;
  const size_t smem = win_bytes + 2 * ((pl.vals_bytes + 127) / 128 * 128);
  auto go = [&](auto kern) {
    GH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    const int64_t items = (int64_t)a.n_tiles * a.n_batches;
    const unsigned blocks =
        static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(items, ctx->num_sms)));
    KTimer kt(ctx, "gather");
    kern<<<blocks, kTopkNW * 32, smem, ctx->stream>>>(a, tk);
    GH_LAUNCHED(ctx);
  };
  const int pq = pl.p4 / 4;
  if (t->P == 16) go(k_gather_topk<16, 4>);
  else if (pq <= 1) go(k_gather_topk<0, 1>);
  else if (pq <= 4) go(k_gather_topk<0, 4>);
  else if (pq <= 8) go(k_gather_topk<0, 8>);
  else go(k_gather_topk<0, 16>);
}

void launch_topk_merge(Ctx* ctx, const unsigned long long* cand_d, int T, int n_lists, int K,
                       int64_t* idx_d, float* val_d) {
  KTimer kt(ctx, "merge");
  k_topk_merge<<<(T + 7) / 8, 256, 0, ctx->stream>>>(cand_d, T, n_lists, K, idx_d, val_d);
  GH_LAUNCHED(ctx);
}

}  // namespace gh

#ifdef GH_TOPK_PROF
extern "C" int gh_topk_prof_read(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_topk_prof, sizeof(g_topk_prof));
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_topk_prof, z, sizeof(z));
  }
  return 0;
}
#endif
