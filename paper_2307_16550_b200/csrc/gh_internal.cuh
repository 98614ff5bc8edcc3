// gh_internal.cuh — shared types and device helpers of the B200 grid-hopping
// library (sm_100a). Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gridhop_b200.h"

namespace gh {

// ------------------------------------------------------------ errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(GH_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define GH_CUDA(x) ::gh::check_cuda((x), #x)
#define GH_LAUNCHED(ctx) \
  do { ::gh::check_cuda(cudaGetLastError(), "kernel launch"); (ctx)->launches++; } while (0)

// ------------------------------------------------------------ host state
struct Buffer {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t n) {
    if (n > bytes) {
      if (p) cudaFree(p);
      p = nullptr;
      bytes = 0;
      GH_CUDA(cudaMalloc(&p, n));
      bytes = n;
    }
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

struct KernelTimes {
  double ms = 0.0;
  int64_t count = 0;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int64_t launches = 0;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  Buffer spectra, frames, keys, misc, twiddle_buf, aprep, mapbuf, seeds, amax, misc2, flagbuf,
      pickctr;
  int twiddle_m = 0;
  int topk_impl = 0;    // 0: auto, 1: fused halo tiles, 2: map then pick, 3: gather + in-loop pick
  int direct_impl = 0;  // 0: tcgen05 3xFP16, 1: CUDA-core fp32, 2: tcgen05 v1, 3: tcgen05 3xTF32
  // host-buffer entry points: copy stream, double-buffer events, pinned staging
  cudaStream_t copy_stream = nullptr;
  bool ev_ready = false;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  void* host_pinned(size_t n) {
    if (n > pinned_bytes) {
      if (pinned) cudaFreeHost(pinned);
      pinned = nullptr;
      pinned_bytes = 0;
      check_cuda(cudaMallocHost(&pinned, n), "cudaMallocHost");
      pinned_bytes = n;
    }
    return pinned;
  }
  // optional per-kernel CUDA-event timing on the context stream
  bool timing = false;
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  std::vector<std::pair<std::string, KernelTimes>> times;
  // deferred campaign-synthesis error flag (window / degenerate geometry)
  int* synth_flag_d = nullptr;
  bool synth_pending = false;
  // bounds-tested kernel builds where one exists (gh_ctx_set_debug_checks)
  bool debug_checks = false;
};

// Records events around one launch when ctx->timing is set.
struct KTimer {
  Ctx* c;
  const char* name;
  cudaEvent_t a = nullptr, b = nullptr;
  static cudaEvent_t take(Ctx* c) {
    if (!c->event_pool.empty()) {
      cudaEvent_t e = c->event_pool.back();
      c->event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  KTimer(Ctx* c_, const char* n) : c(c_), name(n) {
    if (c->timing) {
      a = take(c);
      b = take(c);
      cudaEventRecord(a, c->stream);
    }
  }
  ~KTimer() {
    if (c->timing) {
      cudaEventRecord(b, c->stream);
      c->pending.push_back({name, a, b});
    }
  }
};

// Gather plan: how a CTA stages range windows and walks location bins.
//   full  : every (pair) window is the whole ring; CTAs cover bin chunks.
//   tiled : location tiles (3-D boxes), per-(tile, pair) range windows.
struct TileDesc {
  int32_t x0, y0, z0, wx, wy, wz;
  int64_t entry_off;  // first entry (bin) of this tile in the plan arrays
  int32_t rows;       // staged rows in total (sum over pairs)
  int32_t blk;        // 0: plain order; else 1 + log2 of the 8-bin block's (x, y, z)
                      // extents at bits 0-1, 2-3, 4-5 (extents divide wx, wy, wz)
  // top-K plans: the box above is the tile's core box grown by a 1-bin
  // halo (clipped to the grid); the core (the bins this tile reports) is
  // [c*0, c*0 + cw*) inside it. Other plans: core = box.
  int32_t cx0, cy0, cz0, cwx, cwy, cwz;
};

// values plane pitch (floats) of a top-K tile row: >= wx + 2 (the box plus
// its -inf ring) and == 4 mod 8, so the 4 x 4 positions of a gather step (two
// 2 x 4 entry blocks) store to 16 distinct banks (y * pitch mod 32 =
// 4 * (odd * y mod 8)) and rows stay 16-byte aligned for the LDS.128 filter
__host__ __device__ __forceinline__ int topk_pitch(int wx) {
  return wx + 2 + ((12 - (wx + 2) % 8) % 8);
}
// fused top-K: the kernel's static shared memory (candidate lists, band maxima)
constexpr size_t kTopkListBytes = 8 * 1024;

// Local entry lb of a tile -> tile coordinates. Plain tiles run x-fastest;
// blocked tiles (8-trial power argmax plans) run 8-bin blocks (2 x 4 x 1 on
// 2-D grids, 2 x 1 x 4 on 3-D ones) x-fastest, so a half-warp of the gather
// (8 bins) reads a compact patch: the pairs' rows then advance along two
// axes and spread over the four bank quarters of a 128-byte line instead of
// colliding as a run of 8 bins along x does when a pair's range grows ~2 or
// ~4 rows per bin. A lane's own bins still come in increasing global order.
__host__ __device__ __forceinline__ void tile_local(const TileDesc& td, int64_t lb, int64_t* lx,
                                                    int64_t* ly, int64_t* lz) {
  if (td.blk) {
    const int sx = (td.blk - 1) & 3, sy = ((td.blk - 1) >> 2) & 3, sz = (td.blk - 1) >> 4;
    const int64_t b = lb >> 3, w = lb & 7, nbx = td.wx >> sx, nby = td.wy >> sy;
    *lx = ((b % nbx) << sx) | (w & ((1 << sx) - 1));
    *ly = (((b / nbx) % nby) << sy) | ((w >> sx) & ((1 << sy) - 1));
    *lz = ((b / (nbx * nby)) << sz) | (w >> (sx + sy));
  } else {
    *lx = lb % td.wx;
    *ly = (lb / td.wx) % td.wy;
    *lz = lb / ((int64_t)td.wx * td.wy);
  }
}

// Lane-ordered, bank-complementary entry order of a full-ring plan with
// P <= 3 pairs (permute_for_banks, gh_table.cu). `uniq` are the plan's bins
// in increasing order, par[i] the parity vector of uniq[i]'s ring rows (bit p
// = row parity of pair p). At most 4 complementary couples (v, ~v) exist and
// the gather's 8 lane groups (entry mod 8) form 4 entry pairs: pair class j
// takes its couple's bins in increasing order (entries 8m + 2j, 8m + 2j + 1 =
// the couple's next bin of class v and of class ~v). Every entry pair is
// then bank-complementary and every lane group meets its bins in increasing
// order, so the gather's "first strict maximum" per lane is the smallest bin
// on an exact tie. The bins left when the shortest couple runs out follow in
// ascending order. Appends to *order; returns the first entry of that tail
// (a multiple of 32: the ordered part ends on a gather block).
inline int64_t order_lane_monotone(const std::vector<uint32_t>& uniq,
                                   const std::vector<unsigned>& par, int P,
                                   std::vector<uint32_t>* order) {
  const unsigned full = (1u << P) - 1u;
  std::vector<std::vector<uint32_t>> bucket(static_cast<size_t>(full) + 1);
  for (size_t u = 0; u < uniq.size(); ++u) bucket[par[u] & full].push_back(uniq[u]);
  const int ncpl = 1 << (P - 1), per = 4 / ncpl;
  int64_t steps = INT64_MAX;
  for (int c = 0; c < ncpl; ++c) {
    const size_t n = bucket[c].size() < bucket[full ^ c].size() ? bucket[c].size()
                                                                 : bucket[full ^ c].size();
    const int64_t s = static_cast<int64_t>(n) / per;
    steps = s < steps ? s : steps;
  }
  steps -= steps % 4;
  const size_t base = order->size();
  for (int64_t m = 0; m < steps; ++m)
    for (int j = 0; j < 4; ++j) {
      const int c = j / per;
      const size_t i = static_cast<size_t>(m * per + j % per);
      order->push_back(bucket[c][i]);
      order->push_back(bucket[full ^ c][i]);
    }
  const int64_t tie_from = static_cast<int64_t>(order->size() - base);
  std::vector<uint32_t> rest;
  for (auto& b : bucket)
    for (size_t i = static_cast<size_t>(steps * per); i < b.size(); ++i) rest.push_back(b[i]);
  // ascending (insertion into a sorted run keeps the header free of <algorithm>)
  for (size_t i = 1; i < rest.size(); ++i) {
    const uint32_t x = rest[i];
    size_t k = i;
    for (; k > 0 && rest[k - 1] > x; --k) rest[k] = rest[k - 1];
    rest[k] = x;
  }
  order->insert(order->end(), rest.begin(), rest.end());
  return tie_from;
}

struct Plan {
  bool built = false;
  bool full = false;
  int tb = 16;            // trials per CTA (lanes per bin)
  int esize = 4;          // staged element bytes (float power / float2 complex)
  int k3 = 0;             // 1: consecutive-triple combine with coefficients
  int p4 = 4;             // pairs padded to a multiple of 4 (row array stride)
  int chunk_pairs = 4;    // tiled plan: pairs per staging chunk (own smem region)
  int n_tiles = 0;
  int max_rows = 0;
  TileDesc* tiles_d = nullptr;   // tiled plan
  int4* win_d = nullptr;         // [tiles][P] {base, len, row_start, 0}
  uint16_t* rows_d = nullptr;    // [entries][p4] first staged row per pair
  float2* coef3_d = nullptr;     // [P][3][entries] complex weights (k3, complex schemes)
  float4* coefr_d = nullptr;     // [P][entries] real weights (k3 polar tables), instead of coef3_d
  uint32_t* binid_d = nullptr;   // [entries] global bin of each entry (permuted plans)
  int64_t tie_from = 0;          // permuted plans: first entry of the unordered tail (see permute_for_banks)
  uint32_t* crow_d = nullptr;    // [entries] compact ring rows (cbits per pair), or null
  int cbits = 0;
  int64_t n_entries = 0;
  // top-K plans (halo tiles): per-tile values buffer in shared memory
  bool halo = false;
  size_t vals_bytes = 0;   // [tb trial planes][topk_plane] fp32 values
  int topk_plane = 0;      // floats per trial plane (>= the largest tile's pitch * (wy + 2))
  uint16_t* pos_d = nullptr;  // [entries] values-buffer position of each entry
};

struct Table {
  Ctx* ctx = nullptr;
  int scheme = 1, K = 1;
  int64_t G = 0;              // bins of this table (a shard: layers [slab_lo, slab_hi))
  int64_t bin0 = 0;           // global index of the first bin (location-grid shard)
  int slab_lo = 0, slab_hi = 0;  // layer range along z (3-D) or y (2-D)
  int core_lo = 0, core_hi = 0;  // layers whose peaks top-k reports (halo shards), 0/0: all
  int P = 0, N = 0, os = 1, M = 0;
  double scale = 0.0;
  gh_grid grid{};             // the FULL grid: points stay bit-identical
  std::vector<double> tx, rx;
  double* txrx_d = nullptr;   // [P][6] tx xyz, rx xyz
  uint32_t* idx_d = nullptr;  // [G][P][K]
  double2* coef_d = nullptr;  // [G][P][K]
  double max_residual = 0.0;
  Plan plan;      // argmax gathers (tiled power plans: 8-bin blocked entries)
  Plan plan_map;  // map-mode gathers (plain x-fastest entries: contiguous map stores)
  Plan plan_topk; // fused top-K gathers (halo tiles, values kept in shared memory)
  bool topk_fused_ok = true;  // false once the plan builder found no fused tiling
  int wrap = 1;   // the window policy the table was built with (campaign synthesis)
};

// ------------------------------------------------------------ device helpers
__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__host__ __device__ inline uint64_t substream(uint64_t seed, uint64_t a, uint64_t b) {
  uint64_t x = splitmix64(seed ^ 0x6a09e667f3bcc909ull);
  x = splitmix64(x + 0x9e3779b97f4a7c15ull * (a + 1));
  x = splitmix64(x + 0xbf58476d1ce4e5b9ull * (b + 1));
  return x;
}
__host__ __device__ inline double uniform01(uint64_t key, uint64_t c) {
  const uint64_t v = splitmix64(key + 0x9e3779b97f4a7c15ull * c);
  return static_cast<double>(v >> 11) * 0x1.0p-53;
}
constexpr uint64_t kSceneTag = 0x53434E;

#ifdef __CUDACC__
// Bit-exact restatement of the oracle's norm/sensed_range/grid point: every
// product and sum rounded separately (no FMA contraction).
__device__ inline double dnorm3(const double* a, double x0, double x1, double x2) {
  const double dx = __dsub_rn(x0, a[0]);
  const double dy = __dsub_rn(x1, a[1]);
  const double dz = __dsub_rn(x2, a[2]);
  const double s = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  return __dsqrt_rn(__dadd_rn(s, __dmul_rn(dz, dz)));
}
__device__ inline void dgrid_point(const gh_grid& g, int64_t k, double* o) {
  const int64_t nx = g.n[0], ny = g.n[1];
  const int64_t ix = k % nx, iy = (k / nx) % ny, iz = k / (nx * ny);
  o[0] = __dadd_rn(g.origin[0], __dmul_rn(g.spacing[0], (double)ix));
  o[1] = __dadd_rn(g.origin[1], __dmul_rn(g.spacing[1], (double)iy));
  o[2] = __dadd_rn(g.origin[2], __dmul_rn(g.spacing[2], (double)iz));
}
#endif

// ------------------------------------------------------------ launchers
struct SynthParams {
  const double* txrx_d;  // [P][6]
  double scale;
  gh_campaign camp;
  uint64_t trial0;
  int wrap;
  int* err_flag_d;       // set to 1 on window violation (wrap = 0)
};

// spectra layouts written by the FFT kernel
enum FftOut { FFT_NATURAL = 0, FFT_GATHER_POWER = 1, FFT_GATHER_MAG = 2, FFT_GATHER_COMPLEX = 3 };

void launch_fft(Ctx* ctx, const float2* frames_d, const SynthParams* synth,
                int T, int P, int N, int os, int tb, int out_kind, void* out_d);
// multi-chirp frames: natural spectra [T][P][Mc][M] -> chirp-summed power in
// the gather layout [batch][pair][M][tb]
void launch_chirp_power(Ctx* ctx, const float2* spec_d, int T, int P, int Mc, int M, int tb,
                        float* out_d);
void launch_synth(Ctx* ctx, const SynthParams& sp, int T, int P, int N, float2* frames_d,
                  double* truth_d);
void build_table_device(Ctx* ctx, Table* t, int wrap);
// the gather plan of a table for argmax (mapmode = false) or map-writing
// gathers, built on first use
Plan& build_plan(Ctx* ctx, Table* t, bool mapmode = false);
// the fused top-K plan (2-D K = 1 tiled tables): nullptr when the table does
// not admit one (full-ring / K = 3 / 3-D / shard tables use map + pick)
Plan* build_plan_topk(Ctx* ctx, Table* t);
// fused gather + top-K local maxima: per (trial, tile) candidate keys into
// cand_d [T][n_tiles][K] (thr_d [T] zeroed by the caller), then the merge
void launch_gather_topk(Ctx* ctx, Table* t, const void* spec_d, int T, int K,
                        unsigned long long* cand_d, unsigned long long* thr_d);
// gather + top-K pick with the prune test in the gather loop (gh_gather_pick.cu):
// the argmax plan's tiles, one CTA per 8-trial batch, results straight to
// idx_d / val_d [T][K]
bool gather_pick_ok(const Table* t, const Plan& pl, int K);
void launch_gather_pick(Ctx* ctx, Table* t, const void* spec_d, int T, int K, int64_t* idx_d,
                        float* val_d);
void launch_topk_merge(Ctx* ctx, const unsigned long long* cand_d, int T, int n_lists, int K,
                       int64_t* idx_d, float* val_d);
void launch_gather(Ctx* ctx, Table* t, const void* spec_d, int T, int combine,
                   float* map_d, unsigned long long* keys_d);
void launch_decode_keys(Ctx* ctx, const unsigned long long* keys_d, int T,
                        int64_t* idx_d, float* val_d);
void launch_topk(Ctx* ctx, const float* map_d, int T, const gh_grid& g, int K, int64_t bin0,
                 int64_t* idx_d, float* val_d, int64_t e0 = 0, int64_t e1 = -1);
// velocity stage (gh_velocity.cu): hop (Doppler spectrum lookups) or direct
void launch_velocity(Ctx* ctx, const double* txrx_d, const gh_wave* w, const gh_grid* g,
                     const gh_velocity_grid* vg, const float2* frames_d, int T, int Mc,
                     const int64_t* loc_d, bool hop, int64_t* vidx_d, float* vval_d);
// indirect pipeline, location stage (gh_indirect.cu)
void launch_range_peaks(Ctx* ctx, const float2* spec_d, int64_t rows, int M, int os,
                        double* rhat_d);
void launch_multilaterate(Ctx* ctx, const double* txrx_d, const gh_wave* w, const gh_grid* g,
                          const double* rhat_d, int T, int64_t* idx_d, double* res_d);
// multi-GPU communicator (NCCL, loaded at run time) and the campaign driver
// (gh_campaign.cu)
struct Comm;
void comm_unique_id(uint8_t* id);
Comm* comm_init(Ctx* c, const uint8_t* id, int n_ranks, int rank);
void comm_destroy(Comm* cm);
void comm_info(const Comm* cm, int* n_ranks, int* rank);
void campaign_run(Ctx* c, Comm* comm, const gh_campaign_desc* d, gh_cell_stats* out,
                  int32_t capacity, int32_t* n_cells);
void launch_fit_atoms(Ctx* ctx, int n_samples, int os, const double* r_d, int n, int scheme,
                      uint32_t* idx_d, double2* coef_d, double* res_d);
void launch_add_noise(Ctx* ctx, double2* frames_d, int T, int P, int N, uint64_t seed,
                      uint64_t trial0, double sigma);
// host operations of gh_api.cu used by the campaign driver (gh_campaign.cu)
void op_check_wave(const gh_wave* w);
int64_t op_grid_size(const gh_grid* g);
void op_hop_argmax(Ctx* c, Table* t, const float2* frames, const SynthParams* sp, int T,
                   int combine, int64_t* idx_d, float* val_d);
void op_hop_topk(Ctx* c, Table* t, const float2* frames, const SynthParams* sp, int T, int combine,
                 int K, int64_t* idx_d, float* val_d);
SynthParams op_make_synth(Ctx* c, const double* txrx_d, double scale, const gh_campaign* camp,
                          uint64_t trial0, int wrap);
void op_check_synth(Ctx* c, const SynthParams& sp);
Table* op_new_table(Ctx* c, const gh_wave* w, const gh_grid* g, int scheme);
void op_free_table(Table* t);
void direct_map_simt(Ctx* ctx, const double* txrx_d, const gh_wave* w, const gh_grid* g,
                     const float2* frames_d, int T, int combine, float* map_d,
                     unsigned long long* keys_d);
void direct_map_umma(Ctx* ctx, const double* txrx_d, const gh_wave* w, const gh_grid* g,
                     const float2* frames_d, int T, int combine, float* map_d,
                     unsigned long long* keys_d);
inline void direct_map(Ctx* ctx, const double* txrx_d, const gh_wave* w, const gh_grid* g,
                       const float2* frames_d, int T, int combine, float* map_d,
                       unsigned long long* keys_d) {
  if (ctx->direct_impl == 1)
    direct_map_simt(ctx, txrx_d, w, g, frames_d, T, combine, map_d, keys_d);
  else
    direct_map_umma(ctx, txrx_d, w, g, frames_d, T, combine, map_d, keys_d);
}

}  // namespace gh
