// gh_campaign.cu — the Monte-Carlo campaign driver on the device
// (run_monte_carlo, src/montecarlo.cpp:99-179; hit_ratio / mean_online_ns /
// write_trial_csv / write_summary_csv, montecarlo.cpp:181-284).
//
// Cells run density -> SNR -> algorithm, as the reference's loops do; inside
// a cell this rank's block of trials streams through the device in batches:
// synthesis (fused into the range FFT on the hop arm), the estimator
// (hop argmax / fused top-K, the tcgen05 direct method, or the indirect
// range-peak multilateration), then the statistics kernels — the truths are
// re-drawn from the counter-based scene stream (montecarlo.cpp:48-66), each
// trial's estimates are assigned to its targets and scored (hit ratio per
// threshold, RMSE, half-resolution hits), and the per-trial rows are summed
// in a fixed order into the cell vector. The only host traffic per batch is
// none (CSV records excepted); the only cross-GPU traffic is one NCCL
// all-reduce of the cell vector (sum) and of the cell's device time (max).
// Trials are keyed by (seed, global trial index), so every trial's estimate
// is the same for any rank count (the reference's thread-count invariance,
// tests/test_montecarlo.cpp:125-141).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only: the library is loaded at run time

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <mutex>
#include <string>
#include <vector>

#include "gh_internal.cuh"


namespace gh {
namespace {

// ------------------------------------------------------------ NCCL loader
// dlopen keeps the library loadable on hosts without NCCL; a process that
// already has NCCL (torch's build) shares that copy (RTLD_NOLOAD first).
struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = e ? e : "libnccl.so.2 not found";
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce &&
             api.all_gather && api.error_string;
    if (!api.ok) api.why = "libnccl.so.2 lacks the collectives this library uses";
  });
  if (!api.ok) fail(GH_ERUNTIME, "NCCL not available: " + api.why);
  return api;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(GH_ERUNTIME, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
  int n_ranks = 1, rank = 0, device = 0;
};

namespace {

// ------------------------------------------------------------ kernels

// truths of trials [trial0, trial0 + T): sample_scene's target positions
// (montecarlo.cpp:48-66 + K targets), the draws k_synth makes
__global__ void k_truth(gh_campaign camp, uint64_t trial0, int T, double* truth) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint64_t key = substream(camp.seed, trial0 + (uint64_t)t, kSceneTag);
  const int K = camp.n_targets, D = camp.dims;
  for (int k = 0; k < K; ++k)
    for (int d = 0; d < 3; ++d) {
      double v = camp.area_lo[d];
      if (d < D) {
        const double u = uniform01(key, (uint64_t)(k * D + d));
        v = __dadd_rn(camp.area_lo[d], __dmul_rn(__dsub_rn(camp.area_hi[d], camp.area_lo[d]), u));
      }
      truth[((int64_t)t * K + k) * 3 + d] = v;
    }
}

constexpr int kMaxSlots = 6;        // assignment by permutations: max(kt, ke) <= 6
constexpr int kMaxThresholds = GH_MAX_THRESHOLDS;

struct StatsArgs {
  gh_grid grid;
  const int64_t* est;   // [T][ke] grid bins, -1 = none
  int ke;
  const double* truth;  // [T][kt][3]
  int kt;
  int T;
  double thresholds[kMaxThresholds];
  int nth;
  double half_res, miss_m;
  double* rows;         // [T][ns]: estimates, hits[nth], sum d^2, half-res hits, sum d
  int32_t* assign;      // [T][kt] matched estimate slot (-1 = missed), nullable
};

__device__ bool next_perm(int* a, int n) {
  int i = n - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) return false;
  int j = n - 1;
  while (a[j] <= a[i]) --j;
  const int x = a[i];
  a[i] = a[j];
  a[j] = x;
  for (int l = i + 1, r = n - 1; l < r; ++l, --r) {
    const int y = a[l];
    a[l] = a[r];
    a[r] = y;
  }
  return true;
}

// Restates oracle/gridhop_oracle.cpp or_trial_stats with the same operation
// order (every product / sum rounded separately): one thread per trial.
__global__ void k_trial_stats(StatsArgs a) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.T) return;
  const int n = a.ke > a.kt ? a.ke : a.kt;
  double dist[kMaxSlots][kMaxSlots];
  for (int i = 0; i < a.kt; ++i)
    for (int j = 0; j < n; ++j) {
      const int64_t b = j < a.ke ? a.est[(int64_t)t * a.ke + j] : -1;
      double d = a.miss_m;
      if (b >= 0) {
        double x[3];
        dgrid_point(a.grid, b, x);
        const double* tr = a.truth + ((int64_t)t * a.kt + i) * 3;
        const double dx = __dsub_rn(x[0], tr[0]), dy = __dsub_rn(x[1], tr[1]);
        const double dz = __dsub_rn(x[2], tr[2]);
        d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
      }
      dist[i][j] = d;
    }
  int perm[kMaxSlots], best_p[kMaxSlots];
  for (int j = 0; j < n; ++j) perm[j] = best_p[j] = j;
  double best = 0.0;
  bool have = false;
  do {
    double cost = 0.0;
    for (int i = 0; i < a.kt; ++i) cost = __dadd_rn(cost, __dmul_rn(dist[i][perm[i]], dist[i][perm[i]]));
    if (!have || cost < best) {
      best = cost;
      for (int j = 0; j < n; ++j) best_p[j] = perm[j];
      have = true;
    }
  } while (next_perm(perm, n));
  const int ns = 4 + a.nth;
  double* row = a.rows + (int64_t)t * ns;
  for (int c = 0; c < ns; ++c) row[c] = 0.0;
  for (int i = 0; i < a.kt; ++i) {
    const int j = best_p[i];
    const double d = dist[i][j];
    const bool matched = j < a.ke && a.est[(int64_t)t * a.ke + j] >= 0;
    if (a.assign) a.assign[(int64_t)t * a.kt + i] = matched ? j : -1;
    row[0] += 1.0;
    for (int h = 0; h < a.nth; ++h)
      if (d <= a.thresholds[h]) row[1 + h] += 1.0;
    row[1 + a.nth] = __dadd_rn(row[1 + a.nth], __dmul_rn(d, d));
    if (d <= a.half_res) row[2 + a.nth] += 1.0;
    row[3 + a.nth] = __dadd_rn(row[3 + a.nth], d);
  }
}

// acc[c] += sum over trials of rows[t][c], in a fixed order (thread i sums
// trials i, i + 256, ...; then a fixed tree): deterministic for a batch
__global__ void k_reduce_rows(const double* rows, int T, int ns, double* acc) {
  __shared__ double part[256];
  for (int c = 0; c < ns; ++c) {
    double s = 0.0;
    for (int t = threadIdx.x; t < T; t += 256) s += rows[(int64_t)t * ns + c];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (threadIdx.x < o) part[threadIdx.x] += part[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) acc[c] += part[0];
    __syncthreads();
  }
}

// ------------------------------------------------------------ host helpers

std::string fmt_double(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}
std::string fmt_snr(double snr) { return std::isnan(snr) ? std::string("none") : fmt_double(snr); }
const char* algo_name(int a) {  // algorithm_name (scenario.cpp), enum order of scenario.hpp:12
  return a == GH_ALGO_INDIRECT ? "indirect" : (a == GH_ALGO_DIRECT ? "direct" : "hop");
}

// LocationGrid::build's axis count (model.cpp:91-93) at a density: spacing
// / density over the same extent (n - 1) * spacing from the same origin
gh_grid density_grid(const gh_grid& g, double density) {
  gh_grid o = g;
  for (int d = 0; d < 3; ++d) {
    if (g.n[d] <= 1) continue;
    const double extent = g.spacing[d] * (double)(g.n[d] - 1);
    o.spacing[d] = g.spacing[d] / density;
    o.n[d] = static_cast<int32_t>(std::floor(extent / o.spacing[d] + 1e-9)) + 1;
  }
  return o;
}

struct Record {  // one CSV row source: (trial, algorithm, target)
  int64_t trial;
  int algo;
  int target;
  double truth[3];
  double est[3];  // NaN when the target was missed
};

}  // namespace

void campaign_run(Ctx* c, Comm* comm, const gh_campaign_desc* d, gh_cell_stats* out,
                  int32_t capacity, int32_t* n_cells) {
  if (!d || !n_cells) fail(GH_EINVAL, "campaign: null argument");
  op_check_wave(&d->wave);
  op_grid_size(&d->grid);
  if (d->n_trials < 1) fail(GH_EINVAL, "trials must be >= 1");
  if (d->n_algorithms < 1 || !d->algorithms) fail(GH_EINVAL, "'algorithms' must not be empty");
  for (int i = 0; i < d->n_algorithms; ++i)
    if (d->algorithms[i] < GH_ALGO_INDIRECT || d->algorithms[i] > GH_ALGO_HOP)
      fail(GH_EINVAL, "campaign: unknown algorithm");
  const int topk = d->topk < 1 ? 1 : d->topk;
  if (topk > 8) fail(GH_EINVAL, "top-k: k must be in [1, 8]");
  const int kt = d->scene.n_targets;
  if (kt < 1 || kt > kMaxSlots || topk > kMaxSlots)
    fail(GH_EINVAL, "campaign: statistics assign at most 6 targets / estimates");
  for (int i = 0; i < d->n_algorithms; ++i)
    if (d->algorithms[i] == GH_ALGO_INDIRECT && topk != 1)
      fail(GH_EINVAL, "campaign: the indirect pipeline estimates one location (topk = 1)");
  if (d->combine != GH_POWER && d->combine != GH_MAGNITUDE) fail(GH_EINVAL, "combine: unknown mode");
  std::vector<double> dens = d->n_density > 0 && d->density
                                 ? std::vector<double>(d->density, d->density + d->n_density)
                                 : std::vector<double>{1.0};
  for (double v : dens)
    if (!(std::isfinite(v) && v > 0.0)) fail(GH_EINVAL, "location grid: density must be positive");
  // NaN: a noiseless cell ("none"); no list: the scene's own SNR model
  const bool snr_list = d->n_snr > 0 && d->snr_db;
  std::vector<double> snrs = snr_list ? std::vector<double>(d->snr_db, d->snr_db + d->n_snr)
                                      : std::vector<double>{d->scene.snr_mode == 0
                                                                ? d->scene.snr_db
                                                                : std::nan("")};
  std::vector<double> ths;
  if (d->n_thresholds > 0 && d->thresholds_m) {
    ths.assign(d->thresholds_m, d->thresholds_m + d->n_thresholds);
  } else {
    for (int i = 1; i <= 15; ++i) ths.push_back(0.2 * static_cast<double>(i));  // scenario.cpp:177-179
  }
  if (ths.empty() || ths.size() > kMaxThresholds)
    fail(GH_EINVAL, "campaign: 1 to 32 thresholds");
  const int nth = static_cast<int>(ths.size()), ns = 4 + nth;
  const int n_algo = d->n_algorithms;
  const int64_t cells = (int64_t)dens.size() * snrs.size() * n_algo;
  if (!out || capacity < cells)
    fail(GH_EINVAL, "campaign: output holds fewer cells than density x snr x algorithms");
  *n_cells = 0;
  const int world = comm ? comm->n_ranks : 1, rank = comm ? comm->rank : 0;
  const int64_t base = d->n_trials / world, extra = d->n_trials % world;
  const int64_t lo = rank * base + std::min<int64_t>(rank, extra);
  const int64_t hi = lo + base + (rank < extra ? 1 : 0);
  const int64_t shard_max = base + (extra ? 1 : 0);
  const int P = d->wave.n_pairs, N = d->wave.n_samples, M = N * d->wave.os_range;
  const bool want_csv = d->trial_csv && d->trial_csv[0];
  const double half_res = 0.5 / (2.0 * d->wave.range_scale);  // half of c / (2 B)

  Buffer est_b, val_b, truth_b, rows_b, acc_b, assign_b, frames_b, spec_b, rhat_b, keys_b, map_b,
      flag_b, txrx_b, red_b, gat_b;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  GH_CUDA(cudaEventCreate(&e0));
  GH_CUDA(cudaEventCreate(&e1));
  std::vector<Record> records;
  std::vector<int> cell_of;  // records' cell index
  std::vector<double> cell_online_ns;
  // station coordinates on the device ([P][6]) for direct / indirect
  std::vector<double> h(static_cast<size_t>(P) * 6);
  for (int p = 0; p < P; ++p)
    for (int k = 0; k < 3; ++k) {
      h[static_cast<size_t>(p) * 6 + k] = d->wave.tx[3 * p + k];
      h[static_cast<size_t>(p) * 6 + 3 + k] = d->wave.rx[3 * p + k];
    }
  auto* txrx = static_cast<double*>(txrx_b.get(sizeof(double) * h.size()));
  GH_CUDA(cudaMemcpyAsync(txrx, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, c->stream));
  auto* flag = static_cast<int*>(flag_b.get(sizeof(int)));
  auto* acc = static_cast<double*>(acc_b.get(sizeof(double) * (ns + 1)));

  Table* table = nullptr;
  bool table_owned = true;
  try {
    int cell = 0;
    for (size_t di = 0; di < dens.size(); ++di) {
      const gh_grid grid = density_grid(d->grid, dens[di]);
      const int64_t G = op_grid_size(&grid);
      if (G > 0xffffffffll) fail(GH_EINVAL, "campaign: grid above 2^32 - 1 bins");
      double miss_m = 0.0;
      for (int k = 0; k < 3; ++k) {
        const double e = grid.spacing[k] * (double)grid.n[k];
        miss_m += e * e;
      }
      miss_m = std::sqrt(miss_m);
      double offline_ms = 0.0;
      bool want_hop = false;
      for (int i = 0; i < n_algo; ++i) want_hop |= d->algorithms[i] == GH_ALGO_HOP;
      if (table && table_owned) op_free_table(table);
      table = nullptr;
      bool own_table = true;
      if (want_hop && d->table_source) {  // the caller's TableSource (montecarlo.cpp:125-128)
        int64_t ns_off = 0;
        table = reinterpret_cast<Table*>(d->table_source(d->table_source_user, dens[di], &grid,
                                                         &ns_off));
        if (!table) fail(GH_ERUNTIME, "campaign: the table source returned no table");
        if (table->P != P || table->G != G || table->N != N || table->M != M)
          fail(GH_ERUNTIME, "stale hop table (grid size mismatch)");
        own_table = false;
        offline_ms = (double)ns_off * 1e-6;
      } else if (want_hop) {  // one table per density (montecarlo.cpp:116-136), built on the device
        GH_CUDA(cudaEventRecord(e0, c->stream));
        table = op_new_table(c, &d->wave, &grid, d->scheme);
        table->wrap = d->wrap ? 1 : 0;
        build_table_device(c, table, table->wrap);
        GH_CUDA(cudaEventRecord(e1, c->stream));
        GH_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        GH_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        offline_ms = ms;
      }
      table_owned = own_table;
      for (size_t si = 0; si < snrs.size(); ++si) {
        gh_campaign camp = d->scene;
        if (snr_list) {
          camp.snr_mode = std::isnan(snrs[si]) ? 2 : 0;
          camp.snr_db = std::isnan(snrs[si]) ? 0.0 : snrs[si];
        }
        for (int ai = 0; ai < n_algo; ++ai, ++cell) {
          const int algo = d->algorithms[ai];
          const int ke = topk;
          // batch: hop streams 16k trials (c3 spectra ~4 GB); the direct arm
          // keeps its maps (top-K) under 1 GB
          int64_t B = d->batch > 0 ? d->batch : (algo == GH_ALGO_HOP ? 16384 : 4096);
          if (algo == GH_ALGO_DIRECT && topk > 1)
            B = std::max<int64_t>(1, std::min<int64_t>(B, (int64_t(1) << 28) / G));
          B = std::min<int64_t>(B, std::max<int64_t>(1, hi - lo));
          auto* est = static_cast<int64_t*>(est_b.get(sizeof(int64_t) * B * ke));
          auto* val = static_cast<float*>(val_b.get(sizeof(float) * B * ke));
          auto* truth = static_cast<double*>(truth_b.get(sizeof(double) * B * kt * 3));
          auto* rows = static_cast<double*>(rows_b.get(sizeof(double) * B * ns));
          auto* assign = static_cast<int32_t*>(assign_b.get(sizeof(int32_t) * B * kt));
          GH_CUDA(cudaMemsetAsync(acc, 0, sizeof(double) * (ns + 1), c->stream));
          GH_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), c->stream));
          std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
          std::vector<int64_t> h_est;
          std::vector<int32_t> h_assign;
          std::vector<double> h_truth;
          for (int64_t b0 = lo; b0 < hi; b0 += B) {
            const int nb = static_cast<int>(std::min<int64_t>(B, hi - b0));
            cudaEvent_t ea, eb;
            GH_CUDA(cudaEventCreate(&ea));
            GH_CUDA(cudaEventCreate(&eb));
            evs.push_back({ea, eb});
            if (algo == GH_ALGO_HOP) {
              SynthParams sp = op_make_synth(c, table->txrx_d, table->scale, &camp,
                                             static_cast<uint64_t>(b0), table->wrap);
              sp.err_flag_d = flag;
              // online time: synthesis is fused into the range FFT here
              GH_CUDA(cudaEventRecord(ea, c->stream));
              if (topk > 1) op_hop_topk(c, table, nullptr, &sp, nb, d->combine, topk, est, val);
              else op_hop_argmax(c, table, nullptr, &sp, nb, d->combine, est, val);
              GH_CUDA(cudaEventRecord(eb, c->stream));
            } else {
              SynthParams sp = op_make_synth(c, txrx, d->wave.range_scale, &camp,
                                             static_cast<uint64_t>(b0), d->wrap ? 1 : 0);
              sp.err_flag_d = flag;
              auto* frames = static_cast<float2*>(frames_b.get(sizeof(float2) * nb * P * N));
              launch_synth(c, sp, nb, P, N, frames, nullptr);
              GH_CUDA(cudaEventRecord(ea, c->stream));
              if (algo == GH_ALGO_DIRECT) {
                if (topk == 1) {
                  auto* keys = static_cast<unsigned long long*>(
                      keys_b.get(sizeof(unsigned long long) * nb));
                  GH_CUDA(cudaMemsetAsync(keys, 0, sizeof(unsigned long long) * nb, c->stream));
                  direct_map(c, txrx, &d->wave, &grid, frames, nb, d->combine, nullptr, keys);
                  launch_decode_keys(c, keys, nb, est, val);
                } else {
                  auto* map = static_cast<float*>(map_b.get(sizeof(float) * nb * G));
                  direct_map(c, txrx, &d->wave, &grid, frames, nb, d->combine, map, nullptr);
                  launch_topk(c, map, nb, grid, topk, 0, est, val);
                }
              } else {  // indirect: range peaks + multilateration (indirect.cpp:10-83)
                const int64_t rws = (int64_t)nb * P;
                auto* spec = static_cast<float2*>(spec_b.get(sizeof(float2) * rws * M));
                auto* rh = static_cast<double*>(rhat_b.get(sizeof(double) * rws + sizeof(double) * nb));
                launch_fft(c, frames, nullptr, nb, P, N, d->wave.os_range, 16, FFT_NATURAL, spec);
                launch_range_peaks(c, spec, rws, M, d->wave.os_range, rh);
                launch_multilaterate(c, txrx, &d->wave, &grid, rh, nb, est, rh + rws);
              }
              GH_CUDA(cudaEventRecord(eb, c->stream));
            }
            // statistics of the batch
            k_truth<<<(nb + 127) / 128, 128, 0, c->stream>>>(camp, static_cast<uint64_t>(b0), nb,
                                                             truth);
            GH_LAUNCHED(c);
            StatsArgs sa{};
            sa.grid = grid;
            sa.est = est;
            sa.ke = ke;
            sa.truth = truth;
            sa.kt = kt;
            sa.T = nb;
            for (int i = 0; i < nth; ++i) sa.thresholds[i] = ths[static_cast<size_t>(i)];
            sa.nth = nth;
            sa.half_res = half_res;
            sa.miss_m = miss_m;
            sa.rows = rows;
            sa.assign = assign;
            {
              KTimer kt_(c, "stats");
              k_trial_stats<<<(nb + 127) / 128, 128, 0, c->stream>>>(sa);
              GH_LAUNCHED(c);
              k_reduce_rows<<<1, 256, 0, c->stream>>>(rows, nb, ns, acc);
              GH_LAUNCHED(c);
            }
            if (want_csv) {
              const size_t o_e = h_est.size(), o_a = h_assign.size(), o_t = h_truth.size();
              h_est.resize(o_e + static_cast<size_t>(nb) * ke);
              h_assign.resize(o_a + static_cast<size_t>(nb) * kt);
              h_truth.resize(o_t + static_cast<size_t>(nb) * kt * 3);
              GH_CUDA(cudaMemcpyAsync(h_est.data() + o_e, est, sizeof(int64_t) * nb * ke,
                                      cudaMemcpyDeviceToHost, c->stream));
              GH_CUDA(cudaMemcpyAsync(h_assign.data() + o_a, assign, sizeof(int32_t) * nb * kt,
                                      cudaMemcpyDeviceToHost, c->stream));
              GH_CUDA(cudaMemcpyAsync(h_truth.data() + o_t, truth, sizeof(double) * nb * kt * 3,
                                      cudaMemcpyDeviceToHost, c->stream));
              GH_CUDA(cudaStreamSynchronize(c->stream));
            }
          }
          GH_CUDA(cudaStreamSynchronize(c->stream));
          int hflag = 0;
          GH_CUDA(cudaMemcpy(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost));
          double online = 0.0;
          for (auto& e : evs) {
            float ms = 0.f;
            GH_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
            online += ms;
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
          }
          if (hflag & 2) fail(GH_EDOMAIN, "degenerate geometry: target coincides with a station");
          if (hflag & 1) fail(GH_ERUNTIME, "scene outside unambiguous window");
          // cross-rank: sum of the statistics, max of the device time
          auto* red = static_cast<double*>(red_b.get(sizeof(double)));
          GH_CUDA(cudaMemcpyAsync(red, &online, sizeof(double), cudaMemcpyHostToDevice, c->stream));
          if (comm && comm->n_ranks > 1) {
            check_nccl(nccl().all_reduce(acc, acc, ns, ncclFloat64, ncclSum, comm->comm, c->stream),
                       "ncclAllReduce(stats)");
            check_nccl(nccl().all_reduce(red, red, 1, ncclFloat64, ncclMax, comm->comm, c->stream),
                       "ncclAllReduce(time)");
          }
          std::vector<double> hacc(static_cast<size_t>(ns));
          GH_CUDA(cudaMemcpyAsync(hacc.data(), acc, sizeof(double) * ns, cudaMemcpyDeviceToHost,
                                  c->stream));
          GH_CUDA(cudaMemcpyAsync(&online, red, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
          GH_CUDA(cudaStreamSynchronize(c->stream));
          gh_cell_stats& cs = out[cell];
          std::memset(&cs, 0, sizeof cs);
          cs.algorithm = algo;
          cs.density_idx = static_cast<int32_t>(di);
          cs.snr_idx = static_cast<int32_t>(si);
          cs.n_thresholds = nth;
          cs.density = dens[di];
          cs.snr_db = snrs[si];
          cs.trials = d->n_trials;
          cs.estimates = static_cast<int64_t>(hacc[0]);
          const double cnt = std::max(hacc[0], 1.0);
          for (int i = 0; i < nth; ++i) {
            cs.thresholds_m[i] = ths[static_cast<size_t>(i)];
            cs.hits[i] = hacc[1 + i];
            cs.hit_ratio[i] = hacc[1 + i] / cnt;
          }
          cs.sq_err_sum = hacc[1 + nth];
          cs.hits_half_res = hacc[2 + nth];
          cs.err_sum = hacc[3 + nth];
          cs.rmse_m = std::sqrt(hacc[1 + nth] / cnt);
          cs.online_ms = online;
          cs.offline_ms = algo == GH_ALGO_HOP ? offline_ms : 0.0;
          // the reference times each trial on one thread; here a trial's
          // share of its rank's device time
          cs.mean_online_ns = online * 1e6 / std::max<double>(1.0, (double)shard_max);
          *n_cells = cell + 1;
          if (want_csv) {
            // records of every rank's trials on rank 0: all-gather the
            // estimate / assignment / truth arrays padded to the largest shard
            const int64_t nloc = hi - lo;
            std::vector<double> pack(static_cast<size_t>(shard_max) * kt * 6,
                                     std::nan(""));
            for (int64_t tt = 0; tt < nloc; ++tt)
              for (int i = 0; i < kt; ++i) {
                double* r = &pack[(static_cast<size_t>(tt) * kt + i) * 6];
                for (int k = 0; k < 3; ++k) r[k] = h_truth[(static_cast<size_t>(tt) * kt + i) * 3 + k];
                const int j = h_assign[static_cast<size_t>(tt) * kt + i];
                if (j >= 0) {
                  const int64_t b = h_est[static_cast<size_t>(tt) * ke + j];
                  const int64_t nx = grid.n[0], ny = grid.n[1];
                  const int64_t ix = b % nx, iy = (b / nx) % ny, iz = b / (nx * ny);
                  r[3] = grid.origin[0] + grid.spacing[0] * (double)ix;
                  r[4] = grid.origin[1] + grid.spacing[1] * (double)iy;
                  r[5] = grid.origin[2] + grid.spacing[2] * (double)iz;
                }
              }
            std::vector<double> all;
            if (comm && comm->n_ranks > 1) {
              const size_t per = pack.size();
              auto* g = static_cast<double*>(gat_b.get(sizeof(double) * per * (world + 1)));
              GH_CUDA(cudaMemcpyAsync(g, pack.data(), sizeof(double) * per, cudaMemcpyHostToDevice,
                                      c->stream));
              check_nccl(nccl().all_gather(g, g + per, per, ncclFloat64, comm->comm, c->stream),
                         "ncclAllGather(records)");
              all.resize(per * world);
              GH_CUDA(cudaMemcpyAsync(all.data(), g + per, sizeof(double) * per * world,
                                      cudaMemcpyDeviceToHost, c->stream));
              GH_CUDA(cudaStreamSynchronize(c->stream));
            } else {
              all.swap(pack);
            }
            for (int r = 0; r < world; ++r) {
              const int64_t rlo = r * base + std::min<int64_t>(r, extra);
              const int64_t rn = base + (r < extra ? 1 : 0);
              for (int64_t tt = 0; tt < rn; ++tt)
                for (int i = 0; i < kt; ++i) {
                  const double* q = &all[((static_cast<size_t>(r) * shard_max + tt) * kt + i) * 6];
                  Record rec{rlo + tt, algo, i, {q[0], q[1], q[2]}, {q[3], q[4], q[5]}};
                  records.push_back(rec);
                  cell_of.push_back(cell);
                }
            }
          }
        }
      }
    }
  } catch (...) {
    if (table && table_owned) op_free_table(table);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    throw;
  }
  if (table && table_owned) op_free_table(table);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rank != 0) return;
  if (want_csv) {
    // write_trial_csv (montecarlo.cpp:230-251): record order (density, snr,
    // trial, algorithm), one row per target; Mc = 1 campaigns have no
    // velocity stage (v = 0); a missed target's estimate is NaN
    std::vector<size_t> order(records.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    const int nalg = n_algo;
    std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) {
      const int cx = cell_of[x] / nalg, cy = cell_of[y] / nalg;  // (density, snr)
      if (cx != cy) return cx < cy;
      if (records[x].trial != records[y].trial) return records[x].trial < records[y].trial;
      const int ax = cell_of[x] % nalg, ay = cell_of[y] % nalg;
      if (ax != ay) return ax < ay;
      return records[x].target < records[y].target;
    });
    std::ofstream f(d->trial_csv, std::ios::binary);
    if (!f) fail(GH_ERUNTIME, std::string("cannot write ") + d->trial_csv);
    f << "trial,snr_db,density,algorithm,truth_x0,truth_x1,truth_v0,truth_v1,est_x0,est_x1,"
         "est_v0,est_v1,t_offline_ns,t_online_ns\n";
    for (size_t i : order) {
      const Record& r = records[i];
      const gh_cell_stats& cs = out[cell_of[i]];
      f << r.trial << ',' << fmt_snr(cs.snr_db) << ',' << fmt_double(cs.density) << ','
        << algo_name(r.algo) << ',' << fmt_double(r.truth[0]) << ',' << fmt_double(r.truth[1])
        << ",0,0," << fmt_double(r.est[0]) << ',' << fmt_double(r.est[1]) << ",0,0,"
        << static_cast<int64_t>(cs.offline_ms * 1e6) << ','
        << static_cast<int64_t>(cs.mean_online_ns) << '\n';
    }
    if (!f.flush()) fail(GH_ERUNTIME, std::string("short write: ") + d->trial_csv);
  }
  if (d->summary_csv && d->summary_csv[0]) {
    // write_summary_csv (montecarlo.cpp:253-284): per (density, snr) cell,
    // per algorithm, per threshold
    std::ofstream f(d->summary_csv, std::ios::binary);
    if (!f) fail(GH_ERUNTIME, std::string("cannot write ") + d->summary_csv);
    f << "algorithm,density,snr_db,threshold_m,hit_ratio,mean_online_ns\n";
    for (int i = 0; i < *n_cells; ++i) {
      const gh_cell_stats& cs = out[i];
      for (int h = 0; h < cs.n_thresholds; ++h)
        f << algo_name(cs.algorithm) << ',' << fmt_double(cs.density) << ',' << fmt_snr(cs.snr_db)
          << ',' << fmt_double(cs.thresholds_m[h]) << ',' << fmt_double(cs.hit_ratio[h]) << ','
          << fmt_double(cs.mean_online_ns) << '\n';
    }
    if (!f.flush()) fail(GH_ERUNTIME, std::string("short write: ") + d->summary_csv);
  }
}

}  // namespace gh

// ------------------------------------------------------------ communicator
namespace gh {

void comm_unique_id(uint8_t* id) {
  ncclUniqueId u;
  check_nccl(nccl().get_unique_id(&u), "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof u);
}

Comm* comm_init(Ctx* c, const uint8_t* id, int n_ranks, int rank) {
  if (n_ranks < 1 || rank < 0 || rank >= n_ranks) fail(GH_EINVAL, "comm: bad rank / size");
  NcclApi& api = nccl();
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  auto* cm = new Comm();
  cm->n_ranks = n_ranks;
  cm->rank = rank;
  cm->device = c->device;
  const ncclResult_t r = api.comm_init_rank(&cm->comm, n_ranks, u, rank);
  if (r != ncclSuccess) {
    delete cm;
    fail(GH_ERUNTIME, std::string("ncclCommInitRank: ") + api.error_string(r));
  }
  return cm;
}

void comm_destroy(Comm* cm) {
  if (!cm) return;
  if (cm->comm) nccl().comm_destroy(cm->comm);
  delete cm;
}

void comm_info(const Comm* cm, int* n_ranks, int* rank) {
  *n_ranks = cm->n_ranks;
  *rank = cm->rank;
}

}  // namespace gh
