// gh_gather_pick.cu — BASELINE c3's gather + top-K local-maximum pick with
// no map in HBM and no value planes in shared memory (sm_100a).
//
// The gather is k_gather's (hopping.cpp:59-117 hop_bin_value with Mc = 1:
// 8-trial power rows, one LDS.128 per pair and lane, FADD2); the pick is the
// rule of or_topk_local_max / k_topk_localmax (a bin is a local maximum if
// its value is > every lattice neighbour with a smaller index and >= every
// neighbour with a larger one; candidates rank by value, then by the smaller
// bin: the argmax_index tie rule of src/direct.cpp:55-62).
//
// One CTA owns a batch of 8 trials for the whole grid: it walks the plan's
// tiles one after the other (stage the tile's range windows by TMA bulk
// copies, gather with all 20 warps) and keeps the batch's per-trial top-K
// key lists in shared memory. The gather loop itself only compares each
// value with its trial's prune value — the K-th best local maximum found so
// far, -1 until K are known — which is one FSETP per value, less than the
// argmax update it replaces. A value at or above the prune value is rare
// once the list is full (about K ln G records per trial, plus the bins of
// the peaks' main lobes); the warp then leaves the loop for an out-of-line
// test: lane n evaluates neighbour n of the candidate straight from the
// table's FFT rows and the batch's spectra in global memory (the same fp32
// values added in the same pair order as the gather, so the comparison is
// the map path's bit for bit), and a local maximum enters the trial's list
// under a shared-memory lock. Tiles need no halos and the whole shared
// memory stays with the range windows (the argmax plan's tiles, blocked
// entry order). Batches are handed out by an atomic counter; the trial's
// lists are final when its CTA has walked every tile, so there is no
// candidate buffer and no merge kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <type_traits>

#include "gh_gather_common.cuh"

namespace gh {
namespace {

using namespace ptx;

// 20 warps: 96 registers per thread, so the loop keeps three sets of row words
// (this block and the next two) without spills; 24 warps (80 registers)
// spilled loop invariants and ran 6 % slower, 16 warps 2 % slower
constexpr int kPickThreads = 640;
constexpr int kPickMaxK = 8;
constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kPickQueue = 1024;  // candidate entries per warp queue (global memory)
// CHECK builds (gh_ctx_set_debug_checks): every staged-window offset, window
// extent, queue slot and table / spectra index of the kernel is tested and a
// violation sets one of these bits (compute-sanitizer is closed on this pool)
constexpr unsigned kViolSmemOffset = 1u, kViolQueue = 2u, kViolWindow = 4u, kViolTable = 8u,
                   kViolSpectra = 16u;

struct PickArgs {
  int K;
  const uint32_t* idx;    // table [G][P] FFT rows (K = 1 tables)
  int64_t* out_idx;       // [T][K], -1 = fewer than K maxima
  float* out_val;         // [T][K]
  unsigned* counter;      // batch work counter, zeroed by the launcher
  uint2* queue;           // [CTAs][warps][kPickQueue] candidate queues
  unsigned* viol;         // CHECK builds: bounds-violation mask (see kViol*)
  unsigned smem_bytes;    // CHECK builds: dynamic shared memory of the launch
  int axis3;              // 1: 3-D lattice (26 neighbours, layers along z), 0: 2-D (layers along y)
  int lat_lo, lat_hi;     // layers of the table (a shard holds [lat_lo, lat_hi))
  int core_lo, core_hi;   // layers whose maxima are reported
};

struct __align__(16) PickShared {
  unsigned long long keys[8][kPickMaxK];  // per trial: sorted best keys, 0 = free
  float thr[8];  // per trial: value of the K-th key, -1 until K are known, +inf past T
  int lock[8];
  int batch;
  // what the out-of-line candidate test reads (written once per CTA), so the
  // kernel's parameters never leave the constant bank
  int K, P, M, axis3, nx, ny, nz, lat_lo, lat_hi, core_lo, core_hi;
  int64_t bin0;
  const uint32_t* idx;
  const float* spec;  // the batch's spectra [P][M][8]
  unsigned* viol;     // CHECK builds, else null
  int64_t G;          // bins of the table (CHECK builds)
};

__device__ __forceinline__ uint32_t ord_f(float v) {
  const uint32_t b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// insert key ck into the warp's sorted register list (lane k < K: k-th key)
__device__ __forceinline__ void list_insert(unsigned long long& mine, unsigned long long ck, int K,
                                            int lane) {
  const int pos = __popc(__ballot_sync(kFullMask, lane < K && mine > ck));
  const unsigned long long up = __shfl_up_sync(kFullMask, mine, 1);
  if (lane < K && lane > pos) mine = up;
  if (lane == pos) mine = ck;  // pos < K: ck beats the K-th (or a free slot)
}

// Drain a warp's candidate queue (out of line: nothing of the gather loop is
// live here). An entry is (entry index in the tile | trial slot << 28, value
// bits): a bin whose value reached its trial's prune value and beat its
// neighbours inside its own 2 x 4 entry block. Four candidates at a time
// on 2-D lattices (lane = 8 * candidate + neighbour), one on 3-D ones (26
// neighbours): each tester lane rebuilds its neighbour's value from the
// table's FFT rows and the batch's spectra — the gather's fp32 values added
// in the gather's pair order, so the comparison is the map path's bit for
// bit — and a local maximum enters the trial's list under a lock.
__device__ __noinline__ void drain_candidates(const uint2* q, int qn, const TileDesc* tdp,
                                              PickShared* sh) {
  constexpr int TB = 8;
  const int lane = threadIdx.x & 31;
  const int K = sh->K, P = sh->P, M = sh->M;
  const int nx = sh->nx, ny = sh->ny, nz = sh->nz;
  const bool d3 = sh->axis3 != 0;
  const TileDesc td = *tdp;
  volatile float* thr = sh->thr;
  const int per = d3 ? 1 : 4;             // candidates per round
  const int grp = d3 ? 0 : lane >> 3;     // this lane's candidate of the round
  const int nl = d3 ? lane : lane & 7;    // ... and neighbour
  const int nq = d3 ? (nl < 13 ? nl : nl + 1) : (nl < 4 ? nl : nl + 1);
  const int dx = nq % 3 - 1, dy = (nq / 3) % 3 - 1, dz = d3 ? nq / 9 - 1 : 0;
  const bool tester = d3 ? lane < 26 : true;
  for (int q0 = 0; q0 < qn; q0 += per) {
    const bool have = q0 + grp < qn;
    const uint2 e = have ? q[q0 + grp] : make_uint2(0u, 0u);
    const int ts = (int)(e.x >> 28);
    const float c = __uint_as_float(e.y);
    int64_t lx, ly, lz;
    tile_local(td, (int64_t)(e.x & 0x0fffffffu), &lx, &ly, &lz);
    const int cx = td.x0 + (int)lx, cy = td.y0 + (int)ly, cz = td.z0 + (int)lz;
    const int lay = d3 ? cz : cy;
    const int64_t gb = cx + (int64_t)nx * (cy + (int64_t)ny * cz);
    // stale (the list moved on) or a halo layer (not reported): nothing to test
    const bool want = have && c >= thr[ts] && lay >= sh->core_lo && lay < sh->core_hi;
    const int x = cx + dx, y = cy + dy, z = cz + dz;
    const int nlay = d3 ? z : y;
    bool ok = true;
    bool test = want && tester && x >= 0 && x < nx && y >= 0 && y < ny && z >= 0 && z < nz &&
                nlay >= sh->lat_lo && nlay < sh->lat_hi;
    const int64_t nb = x + (int64_t)nx * (y + (int64_t)ny * z);
    if (test && sh->viol && (nb - sh->bin0 < 0 || nb - sh->bin0 >= sh->G)) {
      atomicOr(sh->viol, kViolTable);
      test = false;
    }
    if (test) {
      const uint32_t* ip = sh->idx + (nb - sh->bin0) * P;
      const float* sp = sh->spec + ts;
      float sum = 0.f;
      // rows, then values, in groups of 16 pairs whose loads fly together
      for (int p0 = 0; p0 < P; p0 += 16) {
        uint32_t row[16];
        float zv[16];
        if (P - p0 >= 16 && (P & 3) == 0) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint4 r4 = __ldg(reinterpret_cast<const uint4*>(ip + p0) + u);
            row[4 * u] = r4.x, row[4 * u + 1] = r4.y, row[4 * u + 2] = r4.z, row[4 * u + 3] = r4.w;
          }
        } else {
#pragma unroll
          for (int u = 0; u < 16; ++u) row[u] = p0 + u < P ? __ldg(ip + p0 + u) : 0u;
        }
        if (sh->viol)
          for (int u = 0; u < 16; ++u)
            if (p0 + u < P && row[u] >= (uint32_t)M) {
              atomicOr(sh->viol, kViolSpectra);
              row[u] = 0u;
            }
#pragma unroll
        for (int u = 0; u < 16; ++u)
          zv[u] = p0 + u < P ? __ldg(sp + ((int64_t)(p0 + u) * M + row[u]) * TB) : 0.f;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (p0 + u < P) sum = p0 + u == 0 ? zv[u] : __fadd_rn(sum, zv[u]);
      }
      ok = nb < gb ? c > sum : c >= sum;
    }
    const unsigned fail = __ballot_sync(kFullMask, !ok);
    for (int g = 0; g < per; ++g) {  // the round's local maxima enter their lists in turn
      const unsigned gmask = d3 ? kFullMask : 0xffu << (8 * g);
      const int src = d3 ? 0 : 8 * g;
      const bool is_max = __shfl_sync(kFullMask, (int)want, src) && !(fail & gmask);
      if (!is_max) continue;  // warp-uniform
      const int gts = __shfl_sync(kFullMask, ts, src);
      const float gc = __shfl_sync(kFullMask, c, src);
      const unsigned long long ggb = __shfl_sync(kFullMask, (unsigned long long)gb, src);
      const unsigned long long key = ((unsigned long long)ord_f(gc) << 32) | (0xffffffffull - ggb);
      if (lane == 0)
        while (atomicCAS(&sh->lock[gts], 0, 1) != 0) {
        }
      __syncwarp();
      __threadfence_block();
      volatile unsigned long long* kl = sh->keys[gts];
      unsigned long long mine = lane < K ? kl[lane] : 0ull;
      const unsigned long long kth = __shfl_sync(kFullMask, mine, K - 1);
      // a seeded maximum meets its bin again in the tile's real pass
      const bool dup = __any_sync(kFullMask, lane < K && mine == key);
      if (key > kth && !dup) {  // warp-uniform
        list_insert(mine, key, K, lane);
        if (lane < K) kl[lane] = mine;
        const unsigned long long nk = __shfl_sync(kFullMask, mine, K - 1);
        if (lane == 0 && nk) thr[gts] = unord_f((uint32_t)(nk >> 32));
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) atomicExch(&sh->lock[gts], 0);
    }
  }
}

// PC: compile-time pair count (0 = runtime, at most 4 * PQ); CHECK: bounds
// tests on every staged offset, window, queue slot and table index
template <int PC, int PQ, bool CHECK = false>
__global__ void __launch_bounds__(kPickThreads, 1) k_gather_pick(GatherArgs a, PickArgs pk) {
  constexpr int TB = 8, ES = 4, L = 2, BPW = 16, NW = kPickThreads / 32;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ PickShared sh;
  __shared__ __align__(8) uint64_t stage_bar;
  const int P = PC ? PC : a.P;
  if (threadIdx.x == 0) {
    mbar_init(&stage_bar, 1);
    mbar_fence_init();
    sh.K = pk.K, sh.P = a.P, sh.M = a.M, sh.axis3 = pk.axis3;
    sh.nx = a.grid.n[0], sh.ny = a.grid.n[1], sh.nz = a.grid.n[2];
    sh.lat_lo = pk.lat_lo, sh.lat_hi = pk.lat_hi, sh.core_lo = pk.core_lo, sh.core_hi = pk.core_hi;
    sh.bin0 = a.bin0;
    sh.idx = pk.idx;
    sh.viol = CHECK ? pk.viol : nullptr;
    sh.G = a.G;
  }
  uint32_t phase = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / L, v = lane % L;
  const float4* smv = reinterpret_cast<const float4*>(smraw) + v;  // this lane's column
  const int pq = PC ? (PC + 3) / 4 : (a.p4 >> 2);                  // uint2 words (4 pairs) per bin
  const uint2* rows2 = reinterpret_cast<const uint2*>(a.rows);
  uint4* sm4 = reinterpret_cast<uint4*>(smraw);
  // this warp's candidate queue (global memory, L2-resident; rarely written):
  // its address is formed where it is used, not kept in registers
  auto my_queue = [&]() { return pk.queue + ((size_t)blockIdx.x * NW + warp) * kPickQueue; };

  for (;;) {
    __syncthreads();  // the previous batch's lists are written out
    if (threadIdx.x == 0) sh.batch = (int)atomicAdd(pk.counter, 1u);
    if (threadIdx.x < TB * kPickMaxK)
      reinterpret_cast<unsigned long long*>(sh.keys)[threadIdx.x] = 0ull;
    __syncthreads();
    const int tb = sh.batch;
    if (tb >= a.n_batches) break;
    if (threadIdx.x < TB) {
      // trials past T (ragged last batch) never become candidates
      sh.thr[threadIdx.x] = tb * TB + (int)threadIdx.x < a.T ? -1.0f : INFINITY;
      sh.lock[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0)
      sh.spec = static_cast<const float*>(a.spec) + (int64_t)tb * a.P * a.M * TB;
    const uint4* spec = reinterpret_cast<const uint4*>(static_cast<const unsigned char*>(a.spec) +
                                                       (int64_t)tb * a.P * a.M * TB * ES);

    // Pass -1 seeds the prune values: tile 0 is gathered once keeping each
    // warp's largest value per trial (the argmax update), and those 20 strip
    // maxima per trial are verified and listed, so the K-th best of them
    // prunes from the first real step on (without it every bin is a
    // candidate until a trial has K maxima). Then every tile, tile 0 again.
    for (int ti = -1; ti < a.n_tiles; ++ti) {
      const int tile = ti < 0 ? 0 : ti;
      const TileDesc* tdp = a.tiles + tile;
      const int64_t entry0 = tdp->entry_off;
      const int nb = tdp->wx * tdp->wy * tdp->wz;
      const int4* win = a.win + (int64_t)tile * a.P;
      __syncthreads();  // the previous tile's readers are done (and sh.thr / sh.spec are set)
      if (warp == 0) {
        // the tile's windows by TMA bulk copies, one pair per lane (the
        // window descriptors load in parallel); then the next tile's windows
        // are asked into L2 so its staging does not wait on HBM
        uint32_t total = 0;
        for (int p = lane; p < P; p += 32) total += (uint32_t)__ldg(&win[p].y) * 16u * L;
        for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(kFullMask, total, o);
        if (lane == 0) mbar_expect_tx(&stage_bar, total);
        __syncwarp();
        for (int p = lane; p < P; p += 32) {
          const int4 w = __ldg(&win[p]);
          if constexpr (CHECK)
            if (w.x < 0 || w.x >= a.M || w.y < 0 || w.y > a.M || w.z < 0 ||
                (size_t)(w.z + w.y) * 16u * L > pk.smem_bytes)
              atomicOr(pk.viol, kViolWindow);
          const uint4* src = spec + (int64_t)p * a.M * L;
          uint4* dst = sm4 + (int64_t)w.z * L;
          for (int r = 0, gi = w.x; r < w.y; gi = 0) {  // base in [0, M): split where it wraps
            const int n = a.M - gi < w.y - r ? a.M - gi : w.y - r;
            bulk_g2s(dst + (int64_t)r * L, src + (int64_t)gi * L, (uint32_t)n * 16u * L,
                     &stage_bar);
            r += n;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&stage_bar);
        if (ti + 1 < a.n_tiles) {
          const int4* nwin = a.win + (int64_t)(ti + 1) * a.P;
          for (int p = lane; p < P; p += 32) {
            const int4 w = __ldg(&nwin[p]);
            const uint4* src = spec + (int64_t)p * a.M * L;
            for (int r = 0, gi = w.x; r < w.y; gi = 0) {
              const int n = a.M - gi < w.y - r ? a.M - gi : w.y - r;
              bulk_prefetch_l2(src + (int64_t)gi * L, (uint32_t)n * 16u * L);
              r += n;
            }
          }
        }
      }
      // 32-entry blocks dealt round-robin to the warps: the bins of a peak's
      // main lobe (a few adjacent blocks, many candidates) spread over
      // several warps' queues instead of making one warp the tile's straggler
      constexpr int kStride = NW * 32;
      const int w0 = warp * 32 < nb ? warp * 32 : nb;
      const int w1 = nb;
      const bool blk24 = tdp->blk == 1 + 1 + (2 << 2);  // 2 x 4 x 1 entry blocks
      // One run over the warp's entries from block `from` until its end or
      // until the queue could overflow in the next block; returns where to
      // resume. The queue is drained between runs, outside the loop, so no
      // call sits among the gather's live registers. SEED (compile time)
      // selects the per-bin action.
      auto run = [&](auto seedc, int from, int& qn) -> int {
        constexpr bool SEED = decltype(seedc)::value;
        uint2 cur[PQ], nxt[PQ], nx2[PQ];  // row words of this block and the next two
        // this lane's row words: word q of entry e at rp[q * ne + e] (32-bit
        // offsets: one base pointer stays live, not one per word)
        const uint2* rp = rows2 + entry0 + lane;
        const unsigned ne = (unsigned)a.n_entries;
#pragma unroll
        for (int q = 0; q < PQ; ++q) cur[q] = nxt[q] = nx2[q] = make_uint2(0u, 0u);
        if (from + lane < w1) {
#pragma unroll
          for (int q = 0; q < PQ; ++q)
            if (q < pq) cur[q] = __ldg(rp + (q * ne + (unsigned)from));
        }
        if (from + kStride + lane < w1) {
#pragma unroll
          for (int q = 0; q < PQ; ++q)
            if (q < pq) nxt[q] = __ldg(rp + (q * ne + (unsigned)(from + kStride)));
        }
        float sbest[4] = {-1.0f, -1.0f, -1.0f, -1.0f};  // SEED: this lane's largest values
        int sblb[4] = {-1, -1, -1, -1};
        // the tile's windows (the first row words load meanwhile; a later run
        // of the same tile finds the phase complete)
        mbar_wait(&stage_bar, phase);
        int blk = from;
        for (; blk < w1; blk += kStride) {
          if (qn > kPickQueue - 256) break;  // a block pushes at most 2 x 32 x 4 entries
          if (blk + 2 * kStride + lane < w1) {  // two blocks ahead: L2 latency under load
#pragma unroll
            for (int q = 0; q < PQ; ++q)
              if (q < pq) nx2[q] = __ldg(rp + (q * ne + (unsigned)(blk + 2 * kStride)));
          }
          float thr[4];
          if constexpr (!SEED)  // one volatile LDS.128: other warps raise these values
            asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(thr[0]), "=f"(thr[1]), "=f"(thr[2]), "=f"(thr[3])
                         : "r"(smem_u32(&sh.thr[v * 4])));
          const int nblk = w1 - blk < 32 ? w1 - blk : 32;
          auto step = [&](int s, bool check) {
            const int j = s * BPW + sub;
            const bool live = !check || j < nblk;
            const int lb = blk + (live ? j : 0);
            float2 acc[2];
            acc[0] = acc[1] = f2(0.f, 0.f);
#pragma unroll
            for (int q = 0; q < PQ; ++q) {
              if (q >= pq) break;
              const unsigned ex = __shfl_sync(kFullMask, cur[q].x, j & 31);
              const unsigned ey = __shfl_sync(kFullMask, cur[q].y, j & 31);
              const unsigned o[4] = {ex & 0xffffu, ex >> 16, ey & 0xffffu, ey >> 16};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int p = 4 * q + u;
                if (PC ? p >= PC : p >= a.P) break;
                if constexpr (CHECK)
                  if (live && (size_t)(o[u] + L) * 16u > (size_t)tdp->rows * 16u * L)
                    atomicOr(pk.viol, kViolSmemOffset);
                accumulate<TB, false, false, L>(smv, o[u], nullptr, acc, p == 0);
              }
            }
            const float vv[4] = {acc[0].x, acc[0].y, acc[1].x, acc[1].y};
            if constexpr (SEED) {
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (live && vv[i] > sbest[i]) {
                  sbest[i] = vv[i];
                  sblb[i] = lb;
                }
            } else {
              const bool hit = live && (vv[0] >= thr[0] || vv[1] >= thr[1] || vv[2] >= thr[2] ||
                                        vv[3] >= thr[3]);
              if (__any_sync(kFullMask, hit)) {
                // rare: queue the candidates. Whole 2 x 4 blocks first drop
                // every bin a neighbour inside its block beats (lane = 2 *
                // (8 * block + 2 * y + x) + v: the neighbour's value is
                // another lane's register; smaller-index neighbours win ties)
                bool cand[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) cand[i] = live && vv[i] >= thr[i];
                if (!check && blk24) {
                  const int w = sub & 7, bx = w & 1, by = w >> 1;
#pragma unroll
                  for (int n = 0; n < 8; ++n) {
                    const int qn_ = n < 4 ? n : n + 1;
                    const int ddx = qn_ % 3 - 1, ddy = qn_ / 3 - 1;
                    const int x2 = bx + ddx, y2 = by + ddy;
                    const bool in = x2 >= 0 && x2 <= 1 && y2 >= 0 && y2 <= 3;
                    const int src = in ? ((((sub & 8) | (y2 * 2 + x2)) << 1) | v) : lane;
                    const bool strict = ddy < 0 || (ddy == 0 && ddx < 0);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                      const float nv = __shfl_sync(kFullMask, vv[i], src);
                      if (in && (strict ? !(vv[i] > nv) : !(vv[i] >= nv))) cand[i] = false;
                    }
                  }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const unsigned m = __ballot_sync(kFullMask, cand[i]);
                  if constexpr (CHECK)
                    if (qn + __popc(m) > kPickQueue) {
                      atomicOr(pk.viol, kViolQueue);
                      continue;
                    }
                  if (cand[i])
                    my_queue()[qn + __popc(m & ((1u << lane) - 1u))] =
                        make_uint2((unsigned)lb | (unsigned)(v * 4 + i) << 28,
                                   __float_as_uint(vv[i]));
                  qn += __popc(m);
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
          for (int q = 0; q < PQ; ++q) {
            cur[q] = nxt[q];
            nxt[q] = nx2[q];
          }
        }
        if constexpr (SEED) {
          // the warp's strip maximum per trial (lanes of equal v share trials)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            for (int o = L; o < 32; o <<= 1) {
              const float ov = __shfl_xor_sync(kFullMask, sbest[i], o);
              const int ol = __shfl_xor_sync(kFullMask, sblb[i], o);
              if (ov > sbest[i] || (ov == sbest[i] && ol >= 0 && (sblb[i] < 0 || ol < sblb[i]))) {
                sbest[i] = ov;
                sblb[i] = ol;
              }
            }
            const bool push = sub == 0 && sblb[i] >= 0 && tb * TB + v * 4 + i < a.T;
            const unsigned m = __ballot_sync(kFullMask, push);
            if (push)
              my_queue()[qn + __popc(m & ((1u << lane) - 1u))] = make_uint2(
                  (unsigned)sblb[i] | (unsigned)(v * 4 + i) << 28, __float_as_uint(sbest[i]));
            qn += __popc(m);
          }
        }
        return blk;
      };
      for (int from = w0;;) {
        int qn = 0;
        from = ti < 0 ? run(std::true_type{}, from, qn) : run(std::false_type{}, from, qn);
        __syncwarp();
        if (qn) drain_candidates(my_queue(), qn, a.tiles + tile, &sh);
        if (from >= w1) break;
      }
      phase ^= 1u;
    }
    __syncthreads();  // every warp's candidates are in the lists
    const int K = pk.K;
    if (threadIdx.x < TB * K) {
      const int ts = threadIdx.x / K, k = threadIdx.x % K;
      const int trial = tb * TB + ts;
      if (trial < a.T) {
        const unsigned long long key = sh.keys[ts][k];
        pk.out_idx[(int64_t)trial * K + k] =
            key ? (int64_t)(0xffffffffull - (key & 0xffffffffull)) : -1;
        pk.out_val[(int64_t)trial * K + k] = key ? unord_f((uint32_t)(key >> 32)) : 0.0f;
      }
    }
  }
}

}  // namespace

bool gather_pick_ok(const Table* t, const Plan& pl, int K) {
  return !pl.full && !pl.k3 && pl.tb == 8 && pl.p4 <= 16 && t->K == 1 && K >= 1 &&
         K <= kPickMaxK;
}

void launch_gather_pick(Ctx* ctx, Table* t, const void* spec_d, int T, int K, int64_t* idx_d,
                        float* val_d) {
  const Plan& pl = t->plan;
  if (!pl.built) fail(GH_ERUNTIME, "gather: plan not built");
  if (!gather_pick_ok(t, pl, K)) fail(GH_EINVAL, "top-k: the pick engine needs a tiled K = 1 plan");
  GatherArgs a{};
  a.spec = spec_d;
  a.tiles = pl.tiles_d;
  a.win = pl.win_d;
  a.rows = pl.rows_d;
  a.n_entries = pl.n_entries;
  a.grid = t->grid;
  a.G = t->G;
  a.bin0 = t->bin0;
  a.P = t->P;
  a.p4 = pl.p4;
  a.M = t->M;
  a.T = T;
  a.n_batches = (T + pl.tb - 1) / pl.tb;
  a.n_tiles = pl.n_tiles;
  PickArgs pk{};
  pk.K = K;
  pk.idx = t->idx_d;
  pk.out_idx = idx_d;
  pk.out_val = val_d;
  const unsigned blocks =
      static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(a.n_batches, ctx->num_sms)));
  // the work counter, then the warps' candidate queues
  auto* scratch = static_cast<unsigned char*>(ctx->pickctr.get(
      256 + sizeof(uint2) * kPickQueue * (kPickThreads / 32) * static_cast<size_t>(ctx->num_sms)));
  pk.counter = reinterpret_cast<unsigned*>(scratch);
  pk.queue = reinterpret_cast<uint2*>(scratch + 256);
  pk.axis3 = t->grid.n[2] > 1 ? 1 : 0;
  pk.lat_lo = t->slab_lo;
  pk.lat_hi = t->slab_hi;
  pk.core_lo = t->core_hi > t->core_lo ? t->core_lo : t->slab_lo;
  pk.core_hi = t->core_hi > t->core_lo ? t->core_hi : t->slab_hi;
  GH_CUDA(cudaMemsetAsync(pk.counter, 0, sizeof(unsigned), ctx->stream));
  const size_t smem = static_cast<size_t>(pl.max_rows) * pl.tb * pl.esize;
  auto go = [&](auto kern) {
    GH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    KTimer kt(ctx, "gather");
    kern<<<blocks, kPickThreads, smem, ctx->stream>>>(a, pk);
    GH_LAUNCHED(ctx);
  };
  const int pq = pl.p4 / 4;
  if (!ctx->debug_checks) {
    if (t->P == 16) go(k_gather_pick<16, 4>);
    else if (pq <= 1) go(k_gather_pick<0, 1>);
    else go(k_gather_pick<0, 4>);
    return;
  }
  // debug build of the same kernel: every shared-memory offset, window,
  // queue slot and table index bounds-tested; synchronous report
  pk.viol = reinterpret_cast<unsigned*>(scratch + 128);
  pk.smem_bytes = static_cast<unsigned>(smem);
  GH_CUDA(cudaMemsetAsync(pk.viol, 0, sizeof(unsigned), ctx->stream));
  if (t->P == 16) go(k_gather_pick<16, 4, true>);
  else if (pq <= 1) go(k_gather_pick<0, 1, true>);
  else go(k_gather_pick<0, 4, true>);
  unsigned mask = 0;
  GH_CUDA(cudaMemcpyAsync(&mask, pk.viol, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
  GH_CUDA(cudaStreamSynchronize(ctx->stream));
  if (mask)
    fail(GH_ERUNTIME, "gather pick: bounds check failed (mask " + std::to_string(mask) +
                          ": 1 staged offset, 2 queue slot, 4 window, 8 table row, 16 spectra row)");
}

}  // namespace gh
