// gh_gather_impl.cuh — the grid-hopping gather-accumulate with fused argmax
// (sm_100a): kernels and launcher, included by gh_gather.cu (K = 1 plans) and
// gh_gather_k3.cu (K = 3 plans), which instantiate one half each.
//
// Reference: hop_bin_value / scan_planes (src/hopping.cpp:59-117):
//   value(bin) = sum_q | sum_j c_j Z_q[I_j(bin, q)] |^2
// with Mc = 1, and argmax_index (src/direct.cpp:55-62, first strict max).
//
// One CTA = (trial batch of TB trials, location tile). It stages the tile's
// per-pair range windows of the batch's spectra into shared memory, layout
// [row][trial]: one TB-run per FFT bin. Lanes are 16-byte vectors: a group
// of L = TB*esize/16 lanes reads one row with LDS.128 (4 trials of power or
// 2 trials of complex spectrum per lane), so a warp serves 32/L bins per
// step; a 128-byte row (32 trials of power, 16 of complex) is exactly one
// shared-memory wavefront, i.e. bank-conflict free.
// The table holds, per (bin, pair), the uint16 shared-memory offset of the
// bin's first row in 16-byte units (row * L), 4 pairs per 64-bit word. It
// streams once per batch of TB trials: each warp owns a contiguous run of
// bins, lane l loads the words of bin l of the next 32-bin block
// (coalesced, one block ahead) and the words reach the lane groups by
// shuffles. Accumulation uses sm_100's packed fp32 adds (FADD2 / FFMA2).
// Argmax is fused: per-lane running max per trial over its bins (increasing
// order, strict >), merged across warps with the smallest-index tie rule,
// then one 64-bit atomicMax per (CTA, trial) on
//   key = float_bits(value) << 32 | (2^32 - 1 - bin)
// which orders by value, then by the smallest bin.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "gh_gather_common.cuh"
#include "gh_internal.cuh"
#include "gh_ptx.cuh"

namespace gh {
namespace {

using namespace ptx;

// threads per CTA (one CTA per SM): 24 warps for power (K = 1) plans, 16
// for the complex K = 3 plans (more registers per thread). Two CTAs per SM
// with half-size windows were measured slower on c3/c4/c5: the windows'
// staging bytes per bin grow faster than the overlap gains.
template <bool K3, bool FULL>
constexpr int gather_threads() { return K3 ? 512 : 768; }

// PLAIN: the plan is known to run x-fastest (map-mode plans), so the
// per-bin map stores skip the blocked-order decode
template <bool PLAIN = false>
__device__ __forceinline__ int64_t global_bin(const GatherArgs& a, const TileDesc& td,
                                              int64_t entry0, int64_t lb) {
  if (a.full) return a.binid ? (int64_t)__ldg(a.binid + entry0 + lb) : a.bin0 + entry0 + lb;
  int64_t lx, ly, lz;
  if (PLAIN) {
    lx = lb % td.wx;
    ly = (lb / td.wx) % td.wy;
    lz = lb / ((int64_t)td.wx * td.wy);
  } else {
    tile_local(td, lb, &lx, &ly, &lz);
  }
  return (td.x0 + lx) + (int64_t)a.grid.n[0] * ((td.y0 + ly) + (int64_t)a.grid.n[1] * (td.z0 + lz));
}

// Exact ties on a bank-permuted full-ring plan. Its ordered part gives every
// lane its bins in increasing order, so the first strict maximum is the
// smallest bin; only a tail entry (a.tie_from on) can tie with a lane's
// running maximum from a larger bin. The gather flags that; here, for the
// flagged trials, the tail entries of the item are re-evaluated from the
// staged ring (same pair order, same adds) and the smallest bin among those
// equal to the item's maximum takes over — argmax_index's first maximum
// (src/direct.cpp:55-62). Out of line: zero frames and noiseless
// mirror-symmetric scenes get here, nothing else.
template <int TB, int L, bool CP, int NT>
__device__ __noinline__ void tail_scan(const uint32_t* crow, const uint16_t* rows,
                                       const uint32_t* binid, int64_t n_entries,
                                       int64_t tie_from, int cbits, int ring, int P,
                                       int64_t entry0, int64_t nb, const float* smf,
                                       unsigned mask, const float* fin_v, unsigned* fin_b) {
  // (plain arguments: a reference to the kernel's parameter struct would
  // force a local copy of it and weigh on the gather loop's registers)
  const int64_t lo = tie_from > entry0 ? tie_from - entry0 : 0;
  for (int64_t job = threadIdx.x; job < (nb - lo) * TB; job += NT) {
    const int tr = (int)(job % TB);
    if (!((mask >> tr) & 1u)) continue;
    const int64_t lb = lo + job / TB;
    float val = 0.f;
    if constexpr (CP) {
      const unsigned wd = __ldg(crow + entry0 + lb);
      const unsigned m = (1u << cbits) - 1u;
      for (int p = 0; p < P; ++p) {
        const unsigned r = (wd >> (cbits * p)) & m;
        const float z = smf[(size_t)((unsigned)(p * ring + r) * L) * 4 + tr];
        val = p == 0 ? z : __fadd_rn(val, z);
      }
    } else {
      for (int p = 0; p < P; ++p) {
        const unsigned o = rows[((int64_t)(p >> 2) * n_entries + entry0 + lb) * 4 + (p & 3)];
        const float z = smf[(size_t)o * 4 + tr];
        val = p == 0 ? z : __fadd_rn(val, z);
      }
    }
    if (val == fin_v[tr]) atomicMin(&fin_b[tr], __ldg(binid + entry0 + lb));
  }
}

// PC: compile-time pair count (0 = runtime, at most 4 * PQ)
// CP (compact rows, full-ring K = 1 plans with P * bits(ring) <= 32): one
// 32-bit word per bin holds every pair's ring row, so a step needs a single
// shuffle instead of two
template <int TB, bool K3, bool MAG, bool MAPMODE, int PC, int PQ, bool FULL, bool CP = false>
__global__ void __launch_bounds__(gather_threads<K3, FULL>(), 1) k_gather(GatherArgs a) {
  constexpr int kGatherThreads = gather_threads<K3, FULL>();
  constexpr int ES = K3 ? 8 : 4;         // staged element bytes
  constexpr int L = TB * ES / 16;        // lanes per row (16 B each)
  constexpr int TPL = 16 / ES;           // trials per lane
  constexpr int BPW = 32 / L;            // bins per warp step
  constexpr int NW = kGatherThreads / 32;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ float red_v[NW * TB];
  __shared__ int red_i[NW * TB];
  __shared__ float fin_v[TB];     // full-ring plans: the item's winners, settled by tail_scan
  __shared__ unsigned fin_b[TB];  // ... their bins
  __shared__ unsigned tie_mask;   // trials whose running maximum tied with a tail entry

  const int P = PC ? PC : a.P;
  __shared__ __align__(8) uint64_t stage_bar;
  if (threadIdx.x == 0) {
    mbar_init(&stage_bar, 1);
    mbar_fence_init();
  }
  uint32_t phase = 0;

  // Work items. Tiled plan: one (location tile = blockIdx.x, trial batch =
  // blockIdx.y) per CTA; tiles of a batch run together, so the batch's
  // spectra stay L2-resident. Full-ring plan: persistent CTAs; the
  // (batch, 32-bin block) space is cut into gridDim.x equal contiguous runs,
  // so every SM does the same work (no tail wave) and restages a ring only
  // where its run enters a new batch.
  int64_t u = 0, u_end = 1, nbpb = 1;
  if constexpr (FULL) {
    nbpb = (a.G + 31) / 32;
    const int64_t U = nbpb * a.n_batches;
    u = U * blockIdx.x / gridDim.x;
    u_end = U * (blockIdx.x + 1) / gridDim.x;
  }
  while (u < u_end) {
  int tb;
  int64_t entry0, nb;
  TileDesc td{};
  const int4* win;
  if constexpr (FULL) {
    tb = static_cast<int>(u / nbpb);
    const int64_t seg_end = (tb + 1) * nbpb < u_end ? (tb + 1) * nbpb : u_end;
    entry0 = (u - tb * nbpb) * 32;
    const int64_t e1 = (seg_end - tb * nbpb) * 32;
    nb = (e1 < a.G ? e1 : a.G) - entry0;
    win = a.win;
    u = seg_end;
  } else {
    tb = blockIdx.y;
    td = a.tiles[blockIdx.x];
    entry0 = td.entry_off;
    nb = (int64_t)td.wx * td.wy * td.wz;
    win = a.win + blockIdx.x * a.P;
    u = u_end;
  }

  // ---- stage the windows: rows (base + r) mod M of every pair. A window is
  // a few contiguous row runs of the batch's spectra (split where it wraps
  // the ring), so the TMA engine copies it with bulk copies while every
  // thread waits on one mbarrier.
  const uint4* spec = reinterpret_cast<const uint4*>(static_cast<const unsigned char*>(a.spec) +
                                                     (int64_t)tb * a.P * a.M * TB * ES);
  uint4* sm4 = reinterpret_cast<uint4*>(smraw);
  __syncthreads();  // barrier initialised / previous item's readers done
  if (threadIdx.x == 0) {
    tie_mask = 0u;  // before the staging it arms: no warp gathers earlier
    uint32_t total = 0;
    for (int p = 0; p < P; ++p) total += (uint32_t)win[p].y * 16u * L;
    mbar_expect_tx(&stage_bar, total);
    for (int p = 0; p < P; ++p) {
      const int4 w = win[p];
      const uint4* src = spec + (int64_t)p * a.M * L;
      uint4* dst = sm4 + (int64_t)w.z * L;
      for (int r = 0, gi = w.x; r < w.y; gi = 0) {  // base in [0, M); K = 3 rings wrap twice
        const int n = a.M - gi < w.y - r ? a.M - gi : w.y - r;
        bulk_g2s(dst + (int64_t)r * L, src + (int64_t)gi * L, (uint32_t)n * 16u * L, &stage_bar);
        r += n;
      }
    }
    mbar_arrive(&stage_bar);
  }

  // ---- gather (the first table block loads while the TMA staging lands)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / L, v = lane % L;
  const float4* smv = reinterpret_cast<const float4*>(smraw) + v;  // this lane's column
  float best[TPL];
  int blb[TPL];
#pragma unroll
  for (int i = 0; i < TPL; ++i) {
    best[i] = -1.0f;
    blb[i] = -1;
  }
  // full plans: 32-entry blocks dealt round-robin to the warps (bank-
  // complementary entry pairs stay on even offsets, a lane still meets its
  // entries in increasing order, and the plan's tail blocks spread over all
  // warps instead of making the last one the straggler); tiled plans:
  // contiguous runs in warp-step multiples, so small tiles still spread over
  // every warp
  constexpr int64_t kRound = BPW;
  const int64_t per_warp = ((nb + NW - 1) / NW + kRound - 1) / kRound * kRound;
  const int64_t w0 = FULL ? warp * 32 : warp * per_warp;
  const int64_t w1 = FULL ? nb : (w0 + per_warp < nb ? w0 + per_warp : nb);
  constexpr int64_t kBlockStep = FULL ? NW * 32 : 32;
  const int pq = PC ? (PC + 3) / 4 : (a.p4 >> 2);  // uint2 words (4 pairs) per bin
  const uint2* rows2 = reinterpret_cast<const uint2*>(a.rows);
  uint2 cur[PQ], nxt[PQ];
#pragma unroll
  for (int q = 0; q < PQ; ++q) {
    cur[q] = make_uint2(0u, 0u);
    nxt[q] = make_uint2(0u, 0u);
  }
  if (w0 + lane < w1) {
    if constexpr (CP) {
      cur[0].x = __ldg(a.crow + entry0 + w0 + lane);
    } else {
#pragma unroll
      for (int q = 0; q < PQ; ++q)
        if (q < pq) cur[q] = __ldg(rows2 + q * a.n_entries + entry0 + w0 + lane);
    }
  }
  mbar_wait(&stage_bar, phase);
  phase ^= 1u;
  // The warp's blocks in two runs of the same loop: the plan's lane-ordered
  // part (TIE = false: exactly the plain gather loop) and, on bank-permuted
  // full plans, its ascending tail from a.tie_from on (TIE = true: the same
  // step plus an equality test that flags exact ties for tail_scan). The
  // row-word prefetch runs across the seam.
  auto blocks = [&](auto tiec, int64_t b0, int64_t b1) -> int64_t {
  constexpr bool TIE = decltype(tiec)::value;
  int64_t blk = b0;
  for (; blk < b1; blk += kBlockStep) {
    unsigned tied = 0u;  // TIE: this lane's trials that met an exact tie in the block
    if (blk + kBlockStep + lane < w1) {
      if constexpr (CP) {
        nxt[0].x = __ldg(a.crow + entry0 + blk + kBlockStep + lane);
      } else {
#pragma unroll
        for (int q = 0; q < PQ; ++q)
          if (q < pq)
            nxt[q] = __ldg(rows2 + q * a.n_entries + entry0 + blk + kBlockStep + lane);
      }
    }
    const int nblk = w1 - blk < 32 ? (int)(w1 - blk) : 32;
    // one step: lane group `sub` handles bin j = s * BPW + sub of the block
    auto step = [&](int s, bool check) {
      const int j = s * BPW + sub;
      const int64_t lb = blk + (!check || j < nblk ? j : 0);
      float2 acc[2];
      acc[0] = acc[1] = f2(0.f, 0.f);
      const float2* cf = K3 && a.coef3 ? a.coef3 + entry0 + lb : nullptr;
      const float4* cr = K3 && a.coefr ? a.coefr + entry0 + lb : nullptr;
      if constexpr (CP) {
        const unsigned wd = __shfl_sync(0xffffffffu, cur[0].x, j & 31);
        const unsigned mask = (1u << a.cbits) - 1u;
#pragma unroll
        for (int p = 0; p < PC; ++p) {
          const unsigned r = (wd >> (a.cbits * p)) & mask;
          accumulate<TB, K3, MAG, L>(smv, (unsigned)(p * a.ring + r) * L, nullptr, acc, p == 0);
        }
      }
#pragma unroll
      for (int q = 0; q < PQ; ++q) {
        if (CP || q >= pq) break;
        const unsigned ex = __shfl_sync(0xffffffffu, cur[q].x, j & 31);
        const unsigned ey = __shfl_sync(0xffffffffu, cur[q].y, j & 31);
        const unsigned o[4] = {ex & 0xffffu, ex >> 16, ey & 0xffffu, ey >> 16};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int p = 4 * q + u;
          if (PC ? p >= PC : p >= a.P) break;
          accumulate<TB, K3, MAG, L>(smv, o[u], cf + 3 * p * a.n_entries, acc, p == 0,
                                     a.n_entries, cr ? cr + p * a.n_entries : nullptr);
        }
      }
      float vals[TPL];
      if constexpr (!K3) {
        vals[0] = acc[0].x;
        vals[1] = acc[0].y;
        vals[2 % TPL] = acc[1].x;
        vals[3 % TPL] = acc[1].y;
      } else {
        vals[0] = acc[0].x;
        vals[1] = acc[0].y;
      }
      if (!check || j < nblk) {
        if constexpr (MAPMODE) {
          const int64_t gb = global_bin<true>(a, td, entry0, lb);
#pragma unroll
          for (int i = 0; i < TPL; ++i) {
            const int trial = tb * TB + v * TPL + i;
            if (trial < a.T) a.map[(int64_t)trial * a.G + (gb - a.bin0)] = vals[i];
          }
        } else {
#pragma unroll
          for (int i = 0; i < TPL; ++i) {
            if (vals[i] > best[i]) {
              best[i] = vals[i];
              blb[i] = (int)lb;
            } else if (TIE && vals[i] == best[i]) {
              // an entry of the plan's unordered tail ties with the lane's
              // running maximum: note the trial, the item's epilogue settles
              // it (tail_scan); only tail blocks test for it
              tied |= 1u << i;
            }
          }
        }
      }
    };
    constexpr bool kUnroll = !K3 && PC > 0 && PC <= 16;
    if (nblk == 32 && kUnroll) {
      // full block: fixed trip count, no bounds checks, fully unrolled so
      // the next step's shuffles and loads overlap this step's updates
#pragma unroll
      for (int s = 0; s < 32 / BPW; ++s) step(s, false);
    } else if (nblk == 32) {
#pragma unroll 1
      for (int s = 0; s < 32 / BPW; ++s) step(s, false);
    } else {
      for (int s = 0; s * BPW < nblk; ++s) step(s, true);
    }
    if constexpr (TIE)
      if (tied) atomicOr(&tie_mask, tied << (v * TPL));
#pragma unroll
    for (int q = 0; q < PQ; ++q) cur[q] = nxt[q];
  }
  return blk;
  };
  if constexpr (FULL && !K3 && !MAPMODE) {
    // tie_from and entry0 are multiples of 32, like every block start
    int64_t wa = a.binid ? a.tie_from - entry0 : w1;
    wa = wa > w1 ? w1 : wa;
    const int64_t seam = blocks(std::false_type{}, w0, wa);  // the warp's first tail block
    blocks(std::true_type{}, seam, w1);
  } else {
    blocks(std::false_type{}, w0, w1);
  }
  if constexpr (!MAPMODE) {
    // exact ties go to the smaller bin: compare global bins (entry order is
    // not bin order on bank-permuted full plans nor in 8-bin blocks)
    auto before = [&](int x, int y) {
      return global_bin(a, td, entry0, x) < global_bin(a, td, entry0, y);
    };
    // merge the BPW lane groups of the warp (same trials, different bins)
#pragma unroll
    for (int i = 0; i < TPL; ++i) {
      for (int o = L; o < 32; o <<= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best[i], o);
        const int oi = __shfl_xor_sync(0xffffffffu, blb[i], o);
        if (oi >= 0 && (blb[i] < 0 || ov > best[i] || (ov == best[i] && before(oi, blb[i])))) {
          best[i] = ov;
          blb[i] = oi;
        }
      }
      if (sub == 0) {
        red_v[warp * TB + v * TPL + i] = best[i];
        red_i[warp * TB + v * TPL + i] = blb[i];
      }
    }
    __syncthreads();
    if (threadIdx.x < TB) {
      float bv = -1.0f;
      int bi = -1;
      for (int w = 0; w < NW; ++w) {
        const float val = red_v[w * TB + threadIdx.x];
        const int i = red_i[w * TB + threadIdx.x];
        if (i < 0) continue;
        if (bi < 0 || val > bv || (val == bv && before(i, bi))) {
          bv = val;
          bi = i;
        }
      }
      const int trial = tb * TB + threadIdx.x;
      const unsigned long long gb =
          bi >= 0 ? (unsigned long long)global_bin(a, td, entry0, bi) : 0ull;
      if constexpr (FULL && !K3) {
        fin_v[threadIdx.x] = bv;
        fin_b[threadIdx.x] = bi >= 0 ? (unsigned)gb : 0xffffffffu;
      } else {
        if (trial < a.T && bi >= 0)
          atomicMax(a.keys + trial, ((unsigned long long)__float_as_uint(bv) << 32) |
                                        (0xffffffffull - gb));
      }
    }
    if constexpr (FULL && !K3) {
      __syncthreads();
      if (tie_mask) {  // CTA-uniform; only degenerate inputs get here
        tail_scan<TB, L, CP, kGatherThreads>(a.crow, a.rows, a.binid, a.n_entries, a.tie_from,
                                             a.cbits, a.ring, P, entry0, nb,
                                             reinterpret_cast<const float*>(smraw), tie_mask,
                                             fin_v, fin_b);
        __syncthreads();
      }
      if (threadIdx.x < TB) {
        const int trial = tb * TB + threadIdx.x;
        if (trial < a.T && fin_b[threadIdx.x] != 0xffffffffu)
          atomicMax(a.keys + trial,
                    ((unsigned long long)__float_as_uint(fin_v[threadIdx.x]) << 32) |
                        (0xffffffffull - (unsigned long long)fin_b[threadIdx.x]));
      }
    }
  }
  }  // work items
}

// ---- tiled plans: persistent CTAs over (tile, trial batch) items, batch
// major so the tiles of a batch run together and its spectra stay
// L2-resident. The windows are staged in pair chunks, each with its own
// shared-memory region and mbarrier: the last warp to finish reading chunk c
// of an item (a shared-memory counter) restages chunk c for the CTA's next
// item right away, so the staging of item i + 1 runs under the gather of
// item i and no warp idles as a producer. Warps walk the pairs chunk by
// chunk with the per-bin sums in registers (up to SMAX warp steps per pass),
// the row words of the next step in flight while the current one
// accumulates; the last chunk finishes each step (argmax or map store).
// CTA warps including the producer: a multiple of 4 so the register file
// splits evenly over the SM sub-partitions (20 warps -> 96 registers, 16 ->
// 128); 20 measured faster than 24 (80 registers, spills) on c5
template <bool K3>
constexpr int tiled_warps() { return K3 ? 16 : 20; }
template <bool K3>
constexpr int tiled_smax() { return K3 ? 6 : 8; }

// issue the bulk copies of chunk c of `item` (one thread; out of line so the
// gather loop keeps its registers)
template <int TB, int ES, int L, int CPP>
__device__ __noinline__ void stage_chunk(const GatherArgs& a, int P, int64_t item, int c,
                                         unsigned char* smraw, uint64_t* bar) {
  int tile, tb;
  item_tile_batch(a, item, &tile, &tb);
  const int4* win = a.win + (int64_t)tile * a.P;
  const uint4* spec = reinterpret_cast<const uint4*>(static_cast<const unsigned char*>(a.spec) +
                                                     (int64_t)tb * a.P * a.M * TB * ES);
  uint4* sm4 = reinterpret_cast<uint4*>(smraw);
  const int p0 = c * CPP, p1 = p0 + CPP < P ? p0 + CPP : P;
  uint32_t total = 0;
  for (int p = p0; p < p1; ++p) total += (uint32_t)__ldg(&win[p].y) * 16u * L;
  mbar_expect_tx(bar, total);
  for (int p = p0; p < p1; ++p) {
    const int4 w = __ldg(&win[p]);
    const uint4* src = spec + (int64_t)p * a.M * L;
    uint4* dst = sm4 + (int64_t)w.z * L;
    for (int r = 0, gi = w.x; r < w.y; gi = 0) {  // K = 3 rings wrap twice
      const int n = a.M - gi < w.y - r ? a.M - gi : w.y - r;
      bulk_g2s(dst + (int64_t)r * L, src + (int64_t)gi * L, (uint32_t)n * 16u * L, bar);
      r += n;
    }
  }
  mbar_arrive(bar);
}

template <int TB, bool K3, bool MAG, bool MAPMODE, int PC, int CQ, int NWT>
__global__ void __launch_bounds__(NWT * 32, 1) k_gather_tiled(GatherArgs a) {
  constexpr int NW = NWT - 1;  // consumer warps; warp NW is the producer
  constexpr int NT = NW * 32;
  constexpr int ES = K3 ? 8 : 4;
  constexpr int L = TB * ES / 16;
  constexpr int TPL = 16 / ES;
  constexpr int BPW = 32 / L;
  constexpr int CPP = 4 * CQ;  // pairs per chunk
  constexpr int SMAX = tiled_smax<K3>();
  constexpr int kMaxChunks = 16;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ float red_v[2][NW * TB];
  __shared__ int red_i[2][NW * TB];
  __shared__ __align__(8) uint64_t full_bar[kMaxChunks], empty_bar[kMaxChunks];
  const int P = PC ? PC : a.P;
  const int NC = (P + CPP - 1) / CPP;
  const int pq = PC ? (PC + 3) / 4 : (a.p4 >> 2);
  const int64_t n_items = (int64_t)a.n_tiles * a.n_batches;
  if (threadIdx.x == 0) {
    for (int c = 0; c < NC; ++c) {
      mbar_init(&full_bar[c], 1);
      mbar_init(&empty_bar[c], NW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == NW) {  // ---- producer: one lane issues the bulk copies
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, ++it)
        for (int c = 0; c < NC; ++c) {
          if (it > 0) mbar_wait(&empty_bar[c], (it - 1) & 1u);
          stage_chunk<TB, ES, L, CPP>(a, P, item, c, smraw, &full_bar[c]);
        }
    }
    return;
  }
  // ---- consumers
  const int sub = lane / L, v = lane % L;
  const float4* smv = reinterpret_cast<const float4*>(smraw) + v;  // this lane's column
  const uint2* rows2 = reinterpret_cast<const uint2*>(a.rows);
  uint32_t it = 0;
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
    int tile, tb;
  item_tile_batch(a, item, &tile, &tb);
    const TileDesc td = a.tiles[tile];
    const int64_t entry0 = td.entry_off;
    const int nb = td.wx * td.wy * td.wz;
    const int per_warp = ((nb + NW - 1) / NW + BPW - 1) / BPW * BPW;
    const int w0 = warp * per_warp < nb ? warp * per_warp : nb;
    const int w1 = w0 + per_warp < nb ? w0 + per_warp : nb;
    const int nsteps = (w1 - w0 + BPW - 1) / BPW;
    const int npass = nsteps > SMAX ? (nsteps + SMAX - 1) / SMAX : 1;
    float best[TPL];
    int blb[TPL];
#pragma unroll
    for (int i = 0; i < TPL; ++i) {
      best[i] = -1.0f;
      blb[i] = -1;
    }
    for (int pass = 0; pass < npass; ++pass) {
      const int sb = w0 + pass * SMAX * BPW;  // first bin of the pass
      float2 acc[SMAX][2];
#pragma unroll
      for (int s = 0; s < SMAX; ++s) acc[s][0] = acc[s][1] = f2(0.f, 0.f);
      for (int c = 0; c < NC; ++c) {
        mbar_wait(&full_bar[c], it & 1u);
        auto load = [&](int s, uint2 (&w)[CQ]) {
          int lb = sb + s * BPW + sub;
          lb = lb < w1 ? lb : w1 - 1;
#pragma unroll
          for (int q = 0; q < CQ; ++q)
            if (c * CQ + q < pq)
              w[q] = __ldg(rows2 + (int64_t)(c * CQ + q) * a.n_entries + entry0 + lb);
        };
        uint2 wc[CQ], wn[CQ];
#pragma unroll
        for (int q = 0; q < CQ; ++q) wc[q] = wn[q] = make_uint2(0u, 0u);
        if (sb < w1) load(0, wc);
#pragma unroll
        for (int s = 0; s < SMAX; ++s) {
          if (sb + s * BPW >= w1) break;  // warp-uniform
          if (s + 1 < SMAX && sb + (s + 1) * BPW < w1) load(s + 1, wn);
          const int lb = sb + s * BPW + sub;
          if (lb < w1) {
            const float2* cf = K3 && a.coef3 ? a.coef3 + entry0 + lb : nullptr;
      const float4* cr = K3 && a.coefr ? a.coefr + entry0 + lb : nullptr;
#pragma unroll
            for (int q = 0; q < CQ; ++q) {
              const unsigned o[4] = {wc[q].x & 0xffffu, wc[q].x >> 16, wc[q].y & 0xffffu,
                                     wc[q].y >> 16};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int p = c * CPP + 4 * q + u;
                if (p >= P) break;
                accumulate<TB, K3, MAG, L>(smv, o[u], cf + 3 * p * a.n_entries, acc[s], false,
                                           a.n_entries, cr ? cr + p * a.n_entries : nullptr);
              }
            }
          }
#pragma unroll
          for (int q = 0; q < CQ; ++q) wc[q] = wn[q];
        }
        if (pass == npass - 1) {  // chunk c of this item fully read
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[c]);
        }
      }
#pragma unroll
      for (int s = 0; s < SMAX; ++s) {  // the pass's bins are complete
        const int lb = sb + s * BPW + sub;
        if (sb + s * BPW >= w1) break;
        if (lb >= w1) continue;
        float vals[TPL];
        if constexpr (!K3) {
          vals[0] = acc[s][0].x;
          vals[1] = acc[s][0].y;
          vals[2 % TPL] = acc[s][1].x;
          vals[3 % TPL] = acc[s][1].y;
        } else {
          vals[0] = acc[s][0].x;
          vals[1] = acc[s][0].y;
        }
        if constexpr (MAPMODE) {
          const int64_t gb = global_bin<true>(a, td, entry0, lb);
#pragma unroll
          for (int i = 0; i < TPL; ++i) {
            const int trial = tb * TB + v * TPL + i;
            if (trial < a.T) a.map[(int64_t)trial * a.G + (gb - a.bin0)] = vals[i];
          }
        } else {
#pragma unroll
          for (int i = 0; i < TPL; ++i)
            if (vals[i] > best[i]) {
              best[i] = vals[i];
              blb[i] = lb;
            }
        }
      }
    }
    if constexpr (!MAPMODE) {
      auto before = [&](int x, int y) {  // exact ties: the smaller bin
        return global_bin(a, td, entry0, x) < global_bin(a, td, entry0, y);
      };
      // merge the warp's lane groups, then the warps (red buffers alternate
      // by item, so one barrier per item suffices)
      float* rv = red_v[it & 1u];
      int* ri = red_i[it & 1u];
#pragma unroll
      for (int i = 0; i < TPL; ++i) {
        for (int o = L; o < 32; o <<= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, best[i], o);
          const int oi = __shfl_xor_sync(0xffffffffu, blb[i], o);
          if (oi >= 0 && (blb[i] < 0 || ov > best[i] || (ov == best[i] && before(oi, blb[i])))) {
            best[i] = ov;
            blb[i] = oi;
          }
        }
        if (sub == 0) {
          rv[warp * TB + v * TPL + i] = best[i];
          ri[warp * TB + v * TPL + i] = blb[i];
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
      if (threadIdx.x < TB) {
        float bv = -1.0f;
        int bi = -1;
        for (int w = 0; w < NW; ++w) {
          const float val = rv[w * TB + threadIdx.x];
          const int i = ri[w * TB + threadIdx.x];
          if (i < 0) continue;
          if (bi < 0 || val > bv || (val == bv && before(i, bi))) {
            bv = val;
            bi = i;
          }
        }
        const int trial = tb * TB + threadIdx.x;
        if (trial < a.T && bi >= 0) {
          const unsigned long long gb = (unsigned long long)global_bin(a, td, entry0, bi);
          atomicMax(a.keys + trial, ((unsigned long long)__float_as_uint(bv) << 32) |
                                        (0xffffffffull - gb));
        }
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

template <int TB, bool K3, bool MAG, bool MAPMODE, int PC, int PQ, bool FULL, bool CP = false>
void run_k(Ctx* ctx, const GatherArgs& a, dim3 grid, size_t smem) {
  constexpr int NT = gather_threads<K3, FULL>();
  auto kern = k_gather<TB, K3, MAG, MAPMODE, PC, PQ, FULL, CP>;
  GH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  if (FULL) {
    // persistent: every resident CTA slot, but >= 4096 bins per CTA so the
    // ring staging stays amortised
    int occ = 0;
    GH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem));
    const int64_t work = a.n_batches * ((a.G + 31) / 32 * 32) / 4096;
    grid = dim3(static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>(work, (int64_t)std::max(occ, 1) * ctx->num_sms))));
  }
  KTimer kt(ctx, "gather");
  kern<<<grid, NT, smem, ctx->stream>>>(a);
  GH_LAUNCHED(ctx);
}

template <int TB, bool K3, bool MAG, bool MAPMODE, int PC, int PQ>
void run(Ctx* ctx, const GatherArgs& a, dim3 grid, size_t smem) {
  if constexpr (TB == 16) {
    if (a.full) {  // full-ring plans are built with 16-trial batches only
      if constexpr (!K3 && !MAPMODE && PC == 3) {
        if (a.crow) {
          run_k<TB, K3, MAG, MAPMODE, PC, PQ, true, true>(ctx, a, grid, smem);
          return;
        }
      }
      run_k<TB, K3, MAG, MAPMODE, PC, PQ, true>(ctx, a, grid, smem);
      return;
    }
  }
  if constexpr (PQ == 16 && TB != 32) {
    if (a.chunk_pairs == 16) {
      // many pairs (17-64): the windows are staging-heavy, so the pipelined
      // persistent kernel (measured 1.6x on BASELINE c5); with <= 16 pairs
      // the stage-then-gather CTAs below measured as fast or faster
      constexpr int NWT = tiled_warps<K3>();
      auto kern = k_gather_tiled<TB, K3, MAG, MAPMODE, PC, 4, NWT>;
      GH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
      int occ = 0;
      GH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NWT * 32, smem));
      const int64_t items = (int64_t)a.n_tiles * a.n_batches;
      const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(
          1, std::min<int64_t>(items, (int64_t)std::max(occ, 1) * ctx->num_sms)));
      KTimer kt(ctx, "gather");
      kern<<<blocks, NWT * 32, smem, ctx->stream>>>(a);
      GH_LAUNCHED(ctx);
      return;
    }
  }
  run_k<TB, K3, MAG, MAPMODE, PC, PQ, false>(ctx, a, grid, smem);
}

// compile-time pair counts of the BASELINE configs (3, 16, 64), runtime
// otherwise (PQ = uint2 words of 4 pairs per bin)
template <int TB, bool K3, bool MAG, bool MAPMODE>
void dispatch_p(Ctx* ctx, const GatherArgs& a, dim3 grid, size_t smem) {
  const int pq = a.p4 / 4;
  if (a.P == 3) run<TB, K3, MAG, MAPMODE, 3, 1>(ctx, a, grid, smem);
  else if (a.P == 16) run<TB, K3, MAG, MAPMODE, 16, 4>(ctx, a, grid, smem);
  else if (a.P == 64) run<TB, K3, MAG, MAPMODE, 64, 16>(ctx, a, grid, smem);
  else if (pq <= 1) run<TB, K3, MAG, MAPMODE, 0, 1>(ctx, a, grid, smem);
  else if (pq <= 4) run<TB, K3, MAG, MAPMODE, 0, 4>(ctx, a, grid, smem);
  else if (pq <= 16) run<TB, K3, MAG, MAPMODE, 0, 16>(ctx, a, grid, smem);
  else fail(GH_EINVAL, "gather: at most 64 TX-RX pairs");
}

template <int TB, bool K3>
void dispatch(Ctx* ctx, const GatherArgs& a, dim3 grid, size_t smem, bool mag, bool mapmode) {
  if (mapmode) {
    if (mag) dispatch_p<TB, K3, true, true>(ctx, a, grid, smem);
    else dispatch_p<TB, K3, false, true>(ctx, a, grid, smem);
  } else {
    if (mag) dispatch_p<TB, K3, true, false>(ctx, a, grid, smem);
    else dispatch_p<TB, K3, false, false>(ctx, a, grid, smem);
  }
}

// The launcher, one side per translation unit: K3SIDE = false instantiates the
// K = 1 (power) kernels (gh_gather.cu), true the K = 3 (complex, interpolation)
// ones (gh_gather_k3.cu) — the two halves compile in parallel.
template <bool K3SIDE>
void launch_gather_side(Ctx* ctx, Table* t, const void* spec_d, int T, int combine, float* map_d,
                        unsigned long long* keys_d) {
  const Plan& pl = map_d ? t->plan_map : t->plan;  // built by the caller (build_plan)
  if (!pl.built) fail(GH_ERUNTIME, "gather: plan not built");
  GatherArgs a{};
  a.spec = spec_d;
  a.tiles = pl.tiles_d;
  a.win = pl.win_d;
  a.rows = pl.rows_d;
  a.n_entries = pl.n_entries;
  a.coef3 = pl.coef3_d;
  a.coefr = pl.coefr_d;
  a.binid = pl.full ? pl.binid_d : nullptr;
  a.crow = pl.full ? pl.crow_d : nullptr;
  a.tie_from = pl.tie_from;
  a.cbits = pl.cbits;
  a.ring = t->M;
  a.grid = t->grid;
  a.G = t->G;
  a.bin0 = t->bin0;
  a.full = pl.full;
  a.P = t->P;
  a.p4 = pl.p4;
  a.M = t->M;
  a.T = T;
  a.map = map_d;
  a.keys = keys_d;
  const int n_tb = (T + pl.tb - 1) / pl.tb;
  a.n_batches = n_tb;
  a.batch_group = 8;  // 64 trials per pass over a tile's plan rows (8-trial batches)
  a.n_tiles = pl.n_tiles;
  a.chunk_pairs = pl.chunk_pairs;
  if (n_tb > 65535) fail(GH_EINVAL, "gather: too many trial batches for one launch");
  const size_t smem = static_cast<size_t>(pl.max_rows) * pl.tb * pl.esize;
  // tiled plan: (tile, batch) CTAs; the full-ring plan's persistent grid is
  // sized in run() from the occupancy
  dim3 grid(pl.full ? 1 : pl.n_tiles, pl.full ? 1 : n_tb);
  const bool mag = combine == GH_MAGNITUDE;
  const bool mapmode = map_d != nullptr;
  if (pl.k3 != K3SIDE) fail(GH_ERUNTIME, "gather: plan / launcher side mismatch");
  if constexpr (!K3SIDE) {
    // K = 1: the FFT epilogue already wrote power or magnitude
    if (pl.tb == 16) dispatch<16, false>(ctx, a, grid, smem, false, mapmode);
    else if (pl.tb == 32) dispatch<32, false>(ctx, a, grid, smem, false, mapmode);
    else if (pl.tb == 8) dispatch<8, false>(ctx, a, grid, smem, false, mapmode);
    else fail(GH_EINVAL, "gather: unsupported trial batch");
  } else {
    if (pl.tb == 16) dispatch<16, true>(ctx, a, grid, smem, mag, mapmode);
    else if (pl.tb == 8) dispatch<8, true>(ctx, a, grid, smem, mag, mapmode);
    else fail(GH_EINVAL, "gather: unsupported trial batch");
  }
}

}  // namespace
}  // namespace gh
