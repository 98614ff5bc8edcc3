// gh_api.cu — the extern "C" boundary (include/gridhop_b200.h).
//
// Every entry point runs its body under `guarded`, which maps gh::Error
// codes (and any other exception) onto the int status + thread-local message
// convention. Validation messages follow the reference's exception texts
// (src/hopping.cpp:17-23, 243-251; src/interp.cpp:156-201; src/model.cpp:50).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>
#include <new>
#include <string>
#include <vector>

#include "gh_internal.cuh"

namespace {

thread_local std::string g_err;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return GH_OK;
  } catch (const gh::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return GH_ERUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GH_ERUNTIME;
  }
}

using gh::fail;

void use_device(gh::Ctx* c) { GH_CUDA(cudaSetDevice(c->device)); }

void check_wave(const gh_wave* w) {
  if (!w) fail(GH_EINVAL, "waveform: null descriptor");
  if (w->n_samples < 2) fail(GH_EINVAL, "waveform: n_samples must be >= 2");
  if (w->os_range < 1) fail(GH_EINVAL, "hop table: oversampling must be >= 1");
  if (!(w->range_scale > 0.0) || !std::isfinite(w->range_scale))
    fail(GH_EINVAL, "waveform: bandwidth must be positive");
  if (w->n_pairs < 1) fail(GH_EINVAL, "geometry: at least one TX-RX pair required");
  if (!w->tx || !w->rx) fail(GH_EINVAL, "geometry: null station arrays");
  for (int i = 0; i < 3 * w->n_pairs; ++i)
    if (!std::isfinite(w->tx[i]) || !std::isfinite(w->rx[i]))
      fail(GH_EINVAL, "geometry: receiver position must be finite");
}

int64_t grid_size(const gh_grid* g) {
  if (!g) fail(GH_EINVAL, "grid: null descriptor");
  for (int d = 0; d < 3; ++d)
    if (g->n[d] < 1) fail(GH_EINVAL, "hop table: empty grid");
  return (int64_t)g->n[0] * g->n[1] * g->n[2];
}

double* upload_txrx(gh::Ctx* c, const gh_wave* w, gh::Buffer& buf) {
  std::vector<double> h(static_cast<size_t>(w->n_pairs) * 6);
  for (int p = 0; p < w->n_pairs; ++p)
    for (int d = 0; d < 3; ++d) {
      h[static_cast<size_t>(p) * 6 + d] = w->tx[3 * p + d];
      h[static_cast<size_t>(p) * 6 + 3 + d] = w->rx[3 * p + d];
    }
  double* d = static_cast<double*>(buf.get(sizeof(double) * h.size()));
  GH_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, c->stream));
  GH_CUDA(cudaStreamSynchronize(c->stream));
  return d;
}

gh::Table* new_table(gh::Ctx* c, const gh_wave* w, const gh_grid* g, int scheme) {
  check_wave(w);
  const int64_t G = grid_size(g);
  if (scheme < GH_NEAREST || scheme > GH_POLAR) fail(GH_EINVAL, "unknown interpolation scheme");
  auto* t = new gh::Table();
  t->ctx = c;
  t->scheme = scheme;
  t->K = scheme == GH_NEAREST ? 1 : (scheme == GH_LINEAR ? 2 : 3);
  t->G = G;
  t->P = w->n_pairs;
  t->N = w->n_samples;
  t->os = w->os_range;
  t->M = w->n_samples * w->os_range;
  t->scale = w->range_scale;
  t->grid = *g;
  t->bin0 = 0;
  t->slab_lo = 0;
  t->slab_hi = g->n[2] > 1 ? g->n[2] : g->n[1];
  t->tx.assign(w->tx, w->tx + 3 * w->n_pairs);
  t->rx.assign(w->rx, w->rx + 3 * w->n_pairs);
  std::vector<double> h(static_cast<size_t>(t->P) * 6);
  for (int p = 0; p < t->P; ++p)
    for (int d = 0; d < 3; ++d) {
      h[static_cast<size_t>(p) * 6 + d] = w->tx[3 * p + d];
      h[static_cast<size_t>(p) * 6 + 3 + d] = w->rx[3 * p + d];
    }
  GH_CUDA(cudaMalloc(&t->txrx_d, sizeof(double) * h.size()));
  GH_CUDA(cudaMemcpy(t->txrx_d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  return t;
}

void free_table(gh::Table* t) {
  if (!t) return;
  cudaFree(t->txrx_d);
  cudaFree(t->idx_d);
  cudaFree(t->coef_d);
  for (gh::Plan* pl : {&t->plan, &t->plan_map, &t->plan_topk}) {
    cudaFree(pl->tiles_d);
    cudaFree(pl->win_d);
    cudaFree(pl->rows_d);
    cudaFree(pl->coef3_d);
    cudaFree(pl->coefr_d);
    cudaFree(pl->binid_d);
    cudaFree(pl->crow_d);
    cudaFree(pl->pos_d);
  }
  delete t;
}

void check_combine(int combine) {
  if (combine != GH_POWER && combine != GH_MAGNITUDE) fail(GH_EINVAL, "combine: unknown mode");
}

// spectra in the gather layout for table t, from frames or from synthesis
// The pick engine hands 8-trial batches to one CTA per SM: its last round is
// only partly filled, so it pays when batches / (rounds * SMs) times its
// measured per-trial advantage over the alternative (c3: 1.5x over map then
// pick, 1.1x over the fused-argmax gather) reaches 1.
bool pick_pays(const gh::Ctx* c, int n_batches, double advantage) {
  if (n_batches < c->num_sms) return false;
  const int rounds = (n_batches + c->num_sms - 1) / c->num_sms;
  return advantage * n_batches >= static_cast<double>(rounds) * c->num_sms;
}

void* gather_spectra(gh::Ctx* c, gh::Table* t, const float2* frames, const gh::SynthParams* sp,
                     int T, int combine, bool mapmode) {
  const gh::Plan& pl = gh::build_plan(c, t, mapmode);
  const int n_tb = (T + pl.tb - 1) / pl.tb;
  const size_t bytes = static_cast<size_t>(n_tb) * t->P * t->M * pl.tb * pl.esize;
  void* spec = c->spectra.get(bytes);
  const int kind = pl.k3 ? gh::FFT_GATHER_COMPLEX
                         : (combine == GH_MAGNITUDE ? gh::FFT_GATHER_MAG : gh::FFT_GATHER_POWER);
  gh::launch_fft(c, frames, sp, T, t->P, t->N, t->os, pl.tb, kind, spec);
  return spec;
}

void hop_argmax(gh::Ctx* c, gh::Table* t, const float2* frames, const gh::SynthParams* sp, int T,
                int combine, int64_t* idx_d, float* val_d) {
  void* spec = gather_spectra(c, t, frames, sp, T, combine, false);
  {
    // The first maximum is the best local maximum (value, then the smaller
    // bin: argmax_index's rule), so where the plan admits the pick engine
    // and there is a batch per SM, its K = 1 form is the faster argmax (one
    // compare per value instead of the compare + two selects; c3: 23.7 vs
    // 26.3 ms per 9,472 trials, identical bins and values). Halo shards keep
    // the plain gather: their argmax covers the halo layers too.
    const gh::Plan& ap = t->plan;
    if (c->topk_impl == 0 && gh::gather_pick_ok(t, ap, 1) && t->core_hi <= t->core_lo &&
        pick_pays(c, (T + ap.tb - 1) / ap.tb, 1.1)) {
      gh::launch_gather_pick(c, t, spec, T, 1, idx_d, val_d);
      return;
    }
  }
  auto* keys = static_cast<unsigned long long*>(c->keys.get(sizeof(unsigned long long) * T));
  GH_CUDA(cudaMemsetAsync(keys, 0, sizeof(unsigned long long) * T, c->stream));
  gh::launch_gather(c, t, spec, T, combine, nullptr, keys);
  gh::launch_decode_keys(c, keys, T, idx_d, val_d);
}

gh::SynthParams make_synth(gh::Ctx* c, const double* txrx_d, double scale, const gh_campaign* camp,
                           uint64_t trial0, int wrap) {
  if (!camp) fail(GH_EINVAL, "campaign: null descriptor");
  if (camp->n_targets < 1 || camp->n_targets > 8)
    fail(GH_EINVAL, "campaign: n_targets must be in [1, 8]");
  if (camp->dims != 2 && camp->dims != 3) fail(GH_EINVAL, "campaign: dims must be 2 or 3");
  if (camp->amp_mode < 0 || camp->amp_mode > 3) fail(GH_EINVAL, "campaign: unknown amp_mode");
  if (camp->snr_mode < 0 || camp->snr_mode > 2) fail(GH_EINVAL, "campaign: unknown snr_mode");
  gh::SynthParams sp{};
  sp.txrx_d = txrx_d;
  sp.scale = scale;
  sp.camp = *camp;
  sp.trial0 = trial0;
  sp.wrap = wrap;
  sp.err_flag_d = static_cast<int*>(c->misc.get(sizeof(int)));
  GH_CUDA(cudaMemsetAsync(sp.err_flag_d, 0, sizeof(int), c->stream));
  return sp;
}

// Campaign synthesis (asynchronous calls): window / geometry violations
// accumulate in a persistent device flag that the next synchronising call
// (gh_ctx_synchronize, gh_campaign_run) reports and clears, so the hot path
// needs no per-step sync (synth.cpp:27-29, model.cpp:50 error texts).
gh::SynthParams make_campaign_synth(gh::Ctx* c, gh::Table* t, const gh_campaign* camp,
                                    uint64_t trial0) {
  gh::SynthParams sp = make_synth(c, t->txrx_d, t->scale, camp, trial0, t->wrap);
  if (!c->synth_flag_d) {
    c->synth_flag_d = static_cast<int*>(c->flagbuf.get(sizeof(int)));
    GH_CUDA(cudaMemsetAsync(c->synth_flag_d, 0, sizeof(int), c->stream));
  }
  sp.err_flag_d = c->synth_flag_d;
  c->synth_pending = true;
  return sp;
}

void check_deferred_synth(gh::Ctx* c) {
  if (!c->synth_pending) return;
  int h = 0;
  GH_CUDA(cudaMemcpyAsync(&h, c->synth_flag_d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  GH_CUDA(cudaMemsetAsync(c->synth_flag_d, 0, sizeof(int), c->stream));
  GH_CUDA(cudaStreamSynchronize(c->stream));
  c->synth_pending = false;
  if (h & 2) fail(GH_EDOMAIN, "degenerate geometry: target coincides with a station");
  if (h & 1) fail(GH_ERUNTIME, "scene outside unambiguous window");
}

void check_synth_flag(gh::Ctx* c, const gh::SynthParams& sp) {
  int h = 0;
  GH_CUDA(cudaMemcpyAsync(&h, sp.err_flag_d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  GH_CUDA(cudaStreamSynchronize(c->stream));
  if (h & 2) fail(GH_EDOMAIN, "degenerate geometry: target coincides with a station");
  if (h & 1) fail(GH_ERUNTIME, "scene outside unambiguous window");
}

// Top-K local maxima per trial (BASELINE c3) through one of three engines
// (below); every engine returns the same lists. The map engine materialises
// the maps of a trial chunk (<= 8 GiB of the 180 GB HBM: ~2000 c3 trials, so
// the FFT and gather launches fill the GPU), then k_topk_localmax picks the
// peaks.
void hop_topk(gh::Ctx* c, gh::Table* t, const float2* frames, const gh::SynthParams* sp, int T,
              int combine, int K, int64_t* idx_d, float* val_d) {
  // Engines (gh_ctx_set_topk_impl): 3 = the gather with the prune test in its
  // loop (gh_gather_pick.cu), 1 = halo tiles with values in shared memory
  // (gh_gather_topk.cu), 2 = map then pick. auto (0) takes engine 3 where the
  // plan admits it and its rounds of one batch per SM are full enough to pay
  // (pick_pays), else 2; every engine returns the same lists.
  if (c->topk_impl == 0 || c->topk_impl == 3) {
    const gh::Plan& ap = gh::build_plan(c, t, false);
    const bool ok = gh::gather_pick_ok(t, ap, K);
    if (c->topk_impl == 3 && !ok)
      fail(GH_EINVAL, "top-k: the pick engine needs a tiled K = 1 plan of at most 16 pairs");
    if (ok && (c->topk_impl == 3 || pick_pays(c, (T + ap.tb - 1) / ap.tb, 1.5))) {
      // trial chunks bound the spectra scratch (~16 GiB of the 180 GB) and
      // split T evenly, so every launch hands each SM many batches
      const int tb = ap.tb;
      const int64_t spec_per_trial = (int64_t)t->P * t->M * ap.esize;
      const int64_t cap = std::max<int64_t>(tb, ((int64_t(1) << 34) / spec_per_trial) / tb * tb);
      const int64_t n_chunks = (T + cap - 1) / cap;
      const int64_t chunk = ((T + n_chunks - 1) / n_chunks + tb - 1) / tb * tb;
      for (int64_t t0 = 0; t0 < T; t0 += chunk) {
        const int tc = static_cast<int>(std::min<int64_t>(chunk, T - t0));
        gh::SynthParams sc{};
        const gh::SynthParams* spc = nullptr;
        if (sp) {
          sc = *sp;
          sc.trial0 += static_cast<uint64_t>(t0);
          spc = &sc;
        }
        const float2* fr = frames ? frames + t0 * t->P * t->N : nullptr;
        void* spec = gather_spectra(c, t, fr, spc, tc, combine, false);
        gh::launch_gather_pick(c, t, spec, tc, K, idx_d + t0 * K, val_d + t0 * K);
      }
      return;
    }
  }
  gh::Plan* tp = c->topk_impl != 1 ? nullptr : gh::build_plan_topk(c, t);
  if (tp) {
    // fused: the gather keeps each tile's values in shared memory and picks
    // the tile's local maxima there; per (trial, tile) K keys, then a merge.
    // Trial chunks bound the spectra (~4 GB) and candidate (~1 GB) scratch.
    const int tb = tp->tb;
    const int64_t n_lists = (int64_t)tp->n_tiles * K;
    const int64_t spec_per_trial = (int64_t)t->P * t->M * tp->esize;
    int64_t chunk = std::min<int64_t>((int64_t(1) << 32) / spec_per_trial,
                                      (int64_t(1) << 30) / (n_lists * 8));
    chunk = std::max<int64_t>(tb, chunk / tb * tb);
    chunk = std::min<int64_t>(chunk, (T + tb - 1) / tb * tb);
    auto* cand = static_cast<unsigned long long*>(
        c->mapbuf.get(sizeof(unsigned long long) * (chunk * n_lists + chunk)));
    unsigned long long* thr = cand + chunk * n_lists;
    for (int t0 = 0; t0 < T; t0 += static_cast<int>(chunk)) {
      const int tc = static_cast<int>(std::min<int64_t>(chunk, T - t0));
      gh::SynthParams sc{};
      const gh::SynthParams* spc = nullptr;
      if (sp) {
        sc = *sp;
        sc.trial0 += static_cast<uint64_t>(t0);
        spc = &sc;
      }
      const float2* fr = frames ? frames + (int64_t)t0 * t->P * t->N : nullptr;
      const size_t bytes = static_cast<size_t>((tc + tb - 1) / tb) * t->P * t->M * tb * tp->esize;
      void* spec = c->spectra.get(bytes);
      gh::launch_fft(c, fr, spc, tc, t->P, t->N, t->os, tb,
                     combine == GH_MAGNITUDE ? gh::FFT_GATHER_MAG : gh::FFT_GATHER_POWER, spec);
      GH_CUDA(cudaMemsetAsync(thr, 0, sizeof(unsigned long long) * tc, c->stream));
      gh::launch_gather_topk(c, t, spec, tc, K, cand, thr);
      gh::launch_topk_merge(c, cand, tc, static_cast<int>(n_lists), K, idx_d + (int64_t)t0 * K,
                            val_d + (int64_t)t0 * K);
    }
    return;
  }
  const int tb = gh::build_plan(c, t, true).tb;
  int64_t chunk = (int64_t(1) << 31) / std::max<int64_t>(t->G, 1);
  chunk = std::max<int64_t>(tb, chunk / tb * tb);
  chunk = std::min<int64_t>(chunk, (T + tb - 1) / tb * tb);
  float* map = static_cast<float*>(c->mapbuf.get(sizeof(float) * chunk * t->G));
  for (int t0 = 0; t0 < T; t0 += static_cast<int>(chunk)) {
    const int tc = static_cast<int>(std::min<int64_t>(chunk, T - t0));
    gh::SynthParams sc{};
    const gh::SynthParams* spc = nullptr;
    if (sp) {
      sc = *sp;
      sc.trial0 += static_cast<uint64_t>(t0);
      spc = &sc;
    }
    const float2* fr = frames ? frames + (int64_t)t0 * t->P * t->N : nullptr;
    void* spec = gather_spectra(c, t, fr, spc, tc, combine, true);
    gh::launch_gather(c, t, spec, tc, combine, map, nullptr);
    // the table's (shard) lattice: its layers only; peaks reported globally
    gh_grid lg = t->grid;
    if (lg.n[2] > 1) lg.n[2] = t->slab_hi - t->slab_lo;
    else lg.n[1] = t->slab_hi - t->slab_lo;
    // halo shards report the peaks of their core layers only; the halo
    // layers complete the border bins' neighbourhoods
    const int64_t layer = (int64_t)lg.n[0] * (lg.n[2] > 1 ? lg.n[1] : 1);
    const int64_t e0 = t->core_hi > t->core_lo ? (t->core_lo - t->slab_lo) * layer : 0;
    const int64_t e1 = t->core_hi > t->core_lo ? (t->core_hi - t->slab_lo) * layer : -1;
    gh::launch_topk(c, map, tc, lg, K, t->bin0, idx_d + (int64_t)t0 * K, val_d + (int64_t)t0 * K,
                    e0, e1);
  }
}

// Multi-chirp location stage (Mc > 1, scan_planes over the slow-time axis,
// hopping.cpp:59-117) for K = 1 tables: per trial chunk, natural spectra of
// every chirp, their power summed over chirps in the gather layout, then the
// unchanged gather (map mode or fused argmax). Chunks keep the natural
// spectra scratch under 4 GiB.
void hop_mc(gh::Ctx* c, gh::Table* t, const float2* frames, int T, int Mc, float* map_d,
            int64_t* idx_d, float* val_d) {
  if (t->K != 1)
    fail(GH_EINVAL, "hop: multi-chirp frames need a K = 1 (nearest) table");
  const gh::Plan& pl = gh::build_plan(c, t, map_d != nullptr);
  const int64_t per_trial = (int64_t)t->P * Mc * t->M;  // complex64 spectra
  int64_t chunk = (int64_t(1) << 29) / std::max<int64_t>(per_trial, 1);
  chunk = std::max<int64_t>(pl.tb, chunk / pl.tb * pl.tb);
  chunk = std::min<int64_t>(chunk, (T + pl.tb - 1) / pl.tb * pl.tb);
  const size_t nat_bytes = sizeof(float2) * per_trial * chunk;
  const size_t pw_bytes = sizeof(float) * (size_t)((chunk + pl.tb - 1) / pl.tb) * pl.tb * t->P * t->M;
  auto* base = static_cast<unsigned char*>(c->spectra.get(nat_bytes + pw_bytes));
  auto* nat = reinterpret_cast<float2*>(base);
  auto* pw = reinterpret_cast<float*>(base + nat_bytes);
  unsigned long long* keys = nullptr;
  if (!map_d) {
    keys = static_cast<unsigned long long*>(c->keys.get(sizeof(unsigned long long) * T));
    GH_CUDA(cudaMemsetAsync(keys, 0, sizeof(unsigned long long) * T, c->stream));
  }
  for (int t0 = 0; t0 < T; t0 += static_cast<int>(chunk)) {
    const int tc = static_cast<int>(std::min<int64_t>(chunk, T - t0));
    // frames [tc][P][Mc][N] are [tc][P*Mc][N]: natural spectra [tc][P][Mc][M]
    gh::launch_fft(c, frames + (int64_t)t0 * t->P * Mc * t->N, nullptr, tc, t->P * Mc, t->N,
                   t->os, 16, gh::FFT_NATURAL, nat);
    gh::launch_chirp_power(c, nat, tc, t->P, Mc, t->M, pl.tb, pw);
    gh::launch_gather(c, t, pw, tc, GH_POWER, map_d ? map_d + (int64_t)t0 * t->G : nullptr,
                      keys ? keys + t0 : nullptr);
  }
  if (!map_d) gh::launch_decode_keys(c, keys, T, idx_d, val_d);
}

__global__ void k_c128_to_c64(const double2* in, float2* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = in[i];
    out[i] = make_float2((float)v.x, (float)v.y);
  }
}


__global__ void k_c64_to_c128(const float2* in, double2* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = in[i];
    out[i] = make_double2((double)v.x, (double)v.y);
  }
}

__global__ void k_f32_to_f64(const float* in, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)in[i];
}

int grid_blocks(int64_t n) { return static_cast<int>(std::min<int64_t>((n + 255) / 256, 148LL * 16)); }

// host complex128 -> device complex64 (scratch `b`, bytes for both forms)
float2* frames_to_device(gh::Ctx* c, gh::Buffer& b, const double* frames, int64_t n) {
  auto* base = static_cast<unsigned char*>(b.get(sizeof(double2) * n + sizeof(float2) * n));
  auto* d128 = reinterpret_cast<double2*>(base);
  auto* d64 = reinterpret_cast<float2*>(base + sizeof(double2) * n);
  GH_CUDA(cudaMemcpyAsync(d128, frames, sizeof(double2) * n, cudaMemcpyHostToDevice, c->stream));
  k_c128_to_c64<<<grid_blocks(n), 256, 0, c->stream>>>(d128, d64, n);
  GH_LAUNCHED(c);
  return d64;
}

// device fp32 values -> host fp64
void values_to_host(gh::Ctx* c, gh::Buffer& b, const float* v_d, int64_t n, double* out) {
  auto* d = static_cast<double*>(b.get(sizeof(double) * n));
  k_f32_to_f64<<<grid_blocks(n), 256, 0, c->stream>>>(v_d, d, n);
  GH_LAUNCHED(c);
  GH_CUDA(cudaMemcpyAsync(out, d, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  GH_CUDA(cudaStreamSynchronize(c->stream));
}

// Host complex128 frames [T][P][N] (the reference's FrameSet element type)
// -> host results [T][k], pipelined over trial chunks: the H2D copy of chunk
// i + 1 (copy stream) overlaps the conversion + estimation of chunk i
// (context stream); each chunk's results are read back as soon as they are
// ready. `run(d64, tc, idx_d, val_d)` estimates one chunk on the device.
template <class Run>
void host_frames_pipeline(gh::Ctx* c, gh::Table* t, const double* frames, int n_trials, int k,
                          int64_t* idx, double* val, Run&& run) {
  const int64_t per = (int64_t)t->P * t->N;
  // ~32 chunks (>= 256 trials each): the copies stream back to back and only
  // the first copy and the last chunk's compute are exposed (measured 8
  // chunks: e2e 528 ms vs the 472 ms PCIe bound on c3; 31 chunks: 486 ms)
  int chunk = n_trials;
  if (n_trials >= 2048) chunk = std::max(256, ((n_trials + 31) / 32 + 255) / 256 * 256);
  // large calls: chunks of whole rounds of one 8-trial batch per SM (what the
  // pick engine hands out), ~80 of them: the exposed first copy and last
  // compute shrink with the chunk (c3: 3,328 -> 1,184 trials per chunk)
  const int unit = 8 * c->num_sms;
  if (chunk > unit) chunk = unit * std::max(1, (n_trials / 80 + unit / 2) / unit);
  const int n_chunks = (n_trials + chunk - 1) / chunk;
  const size_t b128 = sizeof(double2) * per * chunk;
  const int64_t nres = (int64_t)n_trials * k;
  auto* base = static_cast<unsigned char*>(c->frames.get(
      2 * b128 + sizeof(float2) * per * chunk + (sizeof(int64_t) + sizeof(float)) * nres));
  double2* d128[2] = {reinterpret_cast<double2*>(base), reinterpret_cast<double2*>(base + b128)};
  auto* d64 = reinterpret_cast<float2*>(base + 2 * b128);
  auto* didx = reinterpret_cast<int64_t*>(d64 + per * chunk);
  auto* dval = reinterpret_cast<float*>(didx + nres);
  if (!c->copy_stream) GH_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  if (!c->ev_ready) {
    for (int b = 0; b < 2; ++b) {
      GH_CUDA(cudaEventCreateWithFlags(&c->ev_copied[b], cudaEventDisableTiming));
      GH_CUDA(cudaEventCreateWithFlags(&c->ev_consumed[b], cudaEventDisableTiming));
    }
    c->ev_ready = true;
  }
  auto* hpin = static_cast<unsigned char*>(c->host_pinned((sizeof(int64_t) + sizeof(float)) * nres));
  auto* hidx = reinterpret_cast<int64_t*>(hpin);
  auto* hval = reinterpret_cast<float*>(hidx + nres);
  for (int i = 0; i < n_chunks; ++i) {
    const int b = i & 1;
    const int t0 = i * chunk;
    const int tc = std::min(chunk, n_trials - t0);
    const int64_t n = per * tc;
    if (i >= 2) GH_CUDA(cudaStreamWaitEvent(c->copy_stream, c->ev_consumed[b], 0));
    GH_CUDA(cudaMemcpyAsync(d128[b], frames + 2 * per * t0, sizeof(double2) * n,
                            cudaMemcpyHostToDevice, c->copy_stream));
    GH_CUDA(cudaEventRecord(c->ev_copied[b], c->copy_stream));
    GH_CUDA(cudaStreamWaitEvent(c->stream, c->ev_copied[b], 0));
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148LL * 16));
    {
      gh::KTimer kt(c, "convert");
      k_c128_to_c64<<<blocks, 256, 0, c->stream>>>(d128[b], d64, n);
      GH_LAUNCHED(c);
    }
    GH_CUDA(cudaEventRecord(c->ev_consumed[b], c->stream));
    const int64_t r0 = (int64_t)t0 * k;
    run(d64, tc, didx + r0, dval + r0);
    GH_CUDA(cudaMemcpyAsync(hidx + r0, didx + r0, sizeof(int64_t) * tc * k, cudaMemcpyDeviceToHost,
                            c->stream));
    GH_CUDA(cudaMemcpyAsync(hval + r0, dval + r0, sizeof(float) * tc * k, cudaMemcpyDeviceToHost,
                            c->stream));
  }
  GH_CUDA(cudaStreamSynchronize(c->stream));
  std::memcpy(idx, hidx, sizeof(int64_t) * nres);
  for (int64_t i = 0; i < nres; ++i) val[i] = hval[i];
}

// ------------------------------------------------------------ GHT1 container
// Restates save_hop_table / load_hop_table (src/interp.cpp:225-389): the same
// little-endian byte layout and the same runtime_error texts.
constexpr uint32_t kGht1Version = 1;

struct Ght1Reader {
  const char* p;
  size_t left;
  const std::string& path;
  void need(size_t n, const char* what) const {
    if (left < n)
      fail(GH_ERUNTIME, path + ": truncated " + what + " (need " + std::to_string(n) +
                            " bytes, have " + std::to_string(left) + ")");
  }
  template <class T>
  T get(const char* what) {
    need(sizeof(T), what);
    T v;
    std::memcpy(&v, p, sizeof(T));
    p += sizeof(T);
    left -= sizeof(T);
    return v;
  }
};

template <class T>
void ght1_put(std::string& out, T v) {
  out.append(reinterpret_cast<const char*>(&v), sizeof v);
}

std::string ght1_read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(GH_ERUNTIME, path + ": cannot open");
  std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  if (in.bad()) fail(GH_ERUNTIME, path + ": read failed");
  return data;
}

void ght1_write(const std::string& path, const gh_ght1_header& h, const uint32_t* idx,
                const double* coef) {
  if (h.n_pairs < 1 || h.n_bins < 1 || h.k < 1 || h.k > 3 || h.os_range < 1 || h.n_samples < 1)
    fail(GH_EINVAL, "hop table: invalid GHT1 header");
  const size_t entries = (size_t)h.n_bins * (size_t)h.n_pairs * (size_t)h.k;
  std::string out;
  out.reserve(44 + entries * 20);
  out.append("GHT1", 4);
  ght1_put<uint32_t>(out, kGht1Version);
  ght1_put<uint32_t>(out, (uint32_t)h.n_pairs);
  ght1_put<uint32_t>(out, (uint32_t)h.n_bins);
  ght1_put<uint32_t>(out, (uint32_t)h.k);
  ght1_put<uint32_t>(out, (uint32_t)h.os_range);
  ght1_put<uint32_t>(out, (uint32_t)h.n_samples);
  ght1_put<uint64_t>(out, h.scene_hash);
  ght1_put<double>(out, h.max_residual);
  // [bin][pair]: K indices, then K (re, im) — the reference's entry order
  for (size_t e = 0; e < entries; e += (size_t)h.k) {
    for (int j = 0; j < h.k; ++j) ght1_put<uint32_t>(out, idx[e + j]);
    for (int j = 0; j < h.k; ++j) {
      ght1_put<double>(out, coef ? coef[2 * (e + j)] : 1.0);
      ght1_put<double>(out, coef ? coef[2 * (e + j) + 1] : 0.0);
    }
  }
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) fail(GH_ERUNTIME, path + ": cannot open for writing");
  f.write(out.data(), static_cast<std::streamsize>(out.size()));
  f.flush();
  if (!f) fail(GH_ERUNTIME, path + ": short write");
}

// header (+ payload when idx/coef are given: capacity entries)
void ght1_read(const std::string& path, gh_ght1_header& h, uint32_t* idx, double* coef,
               int64_t capacity) {
  const std::string data = ght1_read_file(path);
  Ght1Reader rd{data.data(), data.size(), path};
  rd.need(4, "magic");
  if (std::memcmp(rd.p, "GHT1", 4) != 0)
    fail(GH_ERUNTIME, path + ": bad magic (not a GHT1 hop table)");
  rd.p += 4;
  rd.left -= 4;
  const uint32_t version = rd.get<uint32_t>("version");
  if (version != kGht1Version)
    fail(GH_ERUNTIME, path + ": unsupported hop table version " + std::to_string(version));
  h.n_pairs = (int32_t)rd.get<uint32_t>("receiver count");
  h.n_bins = (int32_t)rd.get<uint32_t>("bin count");
  h.k = (int32_t)rd.get<uint32_t>("order");
  h.os_range = (int32_t)rd.get<uint32_t>("oversampling");
  h.n_samples = (int32_t)rd.get<uint32_t>("sample count");
  h.scene_hash = rd.get<uint64_t>("scene hash");
  h.max_residual = rd.get<double>("worst residual");
  if (h.k < 1 || h.k > 3)
    fail(GH_ERUNTIME, path + ": unsupported interpolation order " + std::to_string(h.k));
  const size_t entries = (size_t)(uint32_t)h.n_bins * (size_t)(uint32_t)h.n_pairs * (size_t)h.k;
  const size_t payload = entries * (4 + 16);
  if (rd.left < payload)
    fail(GH_ERUNTIME, path + ": truncated (expected " + std::to_string(payload) +
                          " payload bytes, have " + std::to_string(rd.left) + ")");
  if (rd.left > payload)
    fail(GH_ERUNTIME, path + ": payload size mismatch (expected " + std::to_string(payload) +
                          " bytes, have " + std::to_string(rd.left) + ")");
  if (!idx && !coef) return;
  if (!idx || !coef || capacity < (int64_t)entries)
    fail(GH_EINVAL, "hop table: GHT1 output arrays too small");
  const uint32_t n_fft = (uint32_t)h.n_samples * (uint32_t)h.os_range;
  for (size_t e = 0; e < entries; e += (size_t)h.k) {
    for (int j = 0; j < h.k; ++j) {
      const uint32_t v = rd.get<uint32_t>("index");
      if (v >= n_fft)
        fail(GH_ERUNTIME, path + ": index " + std::to_string(v) + " outside the FFT grid");
      idx[e + j] = v;
    }
    for (int j = 0; j < h.k; ++j) {
      coef[2 * (e + j)] = rd.get<double>("coefficient");
      coef[2 * (e + j) + 1] = rd.get<double>("coefficient");
    }
  }
}

// ------------------------------------------------------------ MRF1 capture
// Restates write_frames / read_frames (src/frame_io.cpp:53-164) and the
// WaveformConfig / SceneGeometry validation they run (model.cpp:19-43).
constexpr uint32_t kMrf1Version = 1;

void mrf1_validate(const gh_mrf1_header& h, const double* rx) {
  auto check = [](bool ok, const char* what) {
    if (!ok) fail(GH_EINVAL, what);
  };
  check(std::isfinite(h.f0) && h.f0 > 0.0, "waveform: f0 must be positive");
  check(std::isfinite(h.bandwidth) && h.bandwidth > 0.0, "waveform: bandwidth must be positive");
  check(std::isfinite(h.chirp_duration) && h.chirp_duration > 0.0,
        "waveform: chirp_duration must be positive");
  check(h.n_chirps >= 2, "waveform: n_chirps must be >= 2");
  check(h.n_samples >= 2, "waveform: n_samples must be >= 2");
  check(h.n_rx >= 2, "geometry: at least two receivers required");
  for (int i = 0; i < h.n_rx; ++i) {
    check(std::isfinite(rx[2 * i]) && std::isfinite(rx[2 * i + 1]),
          "geometry: receiver position must be finite");
    if (std::hypot(rx[2 * i] - h.tx[0], rx[2 * i + 1] - h.tx[1]) == 0.0)
      fail(GH_EINVAL, "geometry: receiver coincides with TX");
    for (int j = i + 1; j < h.n_rx; ++j)
      if (std::hypot(rx[2 * i] - rx[2 * j], rx[2 * i + 1] - rx[2 * j + 1]) == 0.0)
        fail(GH_EINVAL, "geometry: receivers coincide");
  }
  check(std::isfinite(h.tx[0]) && std::isfinite(h.tx[1]), "geometry: TX position must be finite");
}

// scene_hash (src/model.cpp:135-166), including the reference's offset basis
struct Fnv1a {
  uint64_t h = 1469598103934665603ull;
  void feed(const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) {
      h ^= b[i];
      h *= 1099511628211ull;
    }
  }
  void u32(uint32_t v) { feed(&v, sizeof v); }
  void f64(double v) { feed(&v, sizeof v); }
};

}  // namespace

namespace gh {
// Operations shared with the campaign driver (gh_campaign.cu).
void op_check_wave(const gh_wave* w) { check_wave(w); }
int64_t op_grid_size(const gh_grid* g) { return grid_size(g); }
void op_hop_argmax(Ctx* c, Table* t, const float2* frames, const SynthParams* sp, int T,
                   int combine, int64_t* idx_d, float* val_d) {
  hop_argmax(c, t, frames, sp, T, combine, idx_d, val_d);
}
void op_hop_topk(Ctx* c, Table* t, const float2* frames, const SynthParams* sp, int T, int combine,
                 int K, int64_t* idx_d, float* val_d) {
  hop_topk(c, t, frames, sp, T, combine, K, idx_d, val_d);
}
SynthParams op_make_synth(Ctx* c, const double* txrx_d, double scale, const gh_campaign* camp,
                          uint64_t trial0, int wrap) {
  return make_synth(c, txrx_d, scale, camp, trial0, wrap);
}
void op_check_synth(Ctx* c, const SynthParams& sp) { check_synth_flag(c, sp); }
Table* op_new_table(Ctx* c, const gh_wave* w, const gh_grid* g, int scheme) {
  return new_table(c, w, g, scheme);
}
void op_free_table(Table* t) { free_table(t); }
}  // namespace gh

extern "C" {

const char* gh_last_error(void) { return g_err.c_str(); }
int gh_abi_version(void) { return GH_ABI_VERSION; }

int gh_ctx_create(int32_t device, gh_ctx** out) {
  return guarded([&] {
    if (!out) fail(GH_EINVAL, "ctx: null output");
    int n = 0;
    GH_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) fail(GH_EINVAL, "ctx: no such CUDA device");
    GH_CUDA(cudaSetDevice(device));
    auto* c = new gh::Ctx();
    c->device = device;
    GH_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
    GH_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    int optin = 0;
    GH_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    c->smem_optin = static_cast<size_t>(optin);
    *out = reinterpret_cast<gh_ctx*>(c);
  });
}

int gh_ctx_destroy(gh_ctx* ctx) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    c->spectra.release();
    c->frames.release();
    c->keys.release();
    c->misc.release();
    c->twiddle_buf.release();
    c->aprep.release();
    c->mapbuf.release();
    c->seeds.release();
    c->amax.release();
    c->misc2.release();
    c->flagbuf.release();
    c->pickctr.release();
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->ev_ready)
      for (int b = 0; b < 2; ++b) {
        cudaEventDestroy(c->ev_copied[b]);
        cudaEventDestroy(c->ev_consumed[b]);
      }
    for (auto& p : c->pending) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
  });
}

int gh_ctx_get_stream(gh_ctx* ctx, void** stream) {
  return guarded([&] {
    if (!ctx || !stream) fail(GH_EINVAL, "ctx: null argument");
    *stream = reinterpret_cast<gh::Ctx*>(ctx)->stream;
  });
}

int gh_ctx_set_stream(gh_ctx* ctx, void* stream) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c) fail(GH_EINVAL, "ctx: null argument");
    use_device(c);
    GH_CUDA(cudaStreamSynchronize(c->stream));
    if (c->own_stream) GH_CUDA(cudaStreamDestroy(c->stream));
    c->stream = static_cast<cudaStream_t>(stream);
    c->own_stream = false;
  });
}

int gh_ctx_synchronize(gh_ctx* ctx) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c) fail(GH_EINVAL, "ctx: null argument");
    use_device(c);
    GH_CUDA(cudaStreamSynchronize(c->stream));
    check_deferred_synth(c);
  });
}

int gh_ctx_launch_count(gh_ctx* ctx, int64_t* count) {
  return guarded([&] {
    if (!ctx || !count) fail(GH_EINVAL, "ctx: null argument");
    *count = reinterpret_cast<gh::Ctx*>(ctx)->launches;
  });
}

int gh_ctx_set_direct_impl(gh_ctx* ctx, int32_t impl) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c) fail(GH_EINVAL, "ctx: null argument");
    if (impl < 0 || impl > 4)
      fail(GH_EINVAL,
           "ctx: direct impl must be 0 (tcgen05 3xFP16), 1 (simt), 2 (tcgen05 v1), 3 (tcgen05 "
           "3xTF32) or 4 (tcgen05 1xFP16 fast mode)");
    c->direct_impl = impl;
  });
}

int gh_ctx_set_topk_impl(gh_ctx* ctx, int32_t impl) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c) fail(GH_EINVAL, "ctx: null argument");
    if (impl < 0 || impl > 3)
      fail(GH_EINVAL,
           "ctx: top-k impl must be 0 (auto), 1 (fused halo tiles), 2 (map then pick) or 3 "
           "(gather + in-loop pick)");
    c->topk_impl = impl;
  });
}

int gh_ctx_set_debug_checks(gh_ctx* ctx, int32_t on) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c) fail(GH_EINVAL, "ctx: null argument");
    c->debug_checks = on != 0;
  });
}

int gh_ctx_set_timing(gh_ctx* ctx, int32_t on) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c) fail(GH_EINVAL, "ctx: null argument");
    c->timing = on != 0;
  });
}

int gh_ctx_kernel_time(gh_ctx* ctx, const char* name, double* total_ms, int64_t* count) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || !name) fail(GH_EINVAL, "ctx: null argument");
    use_device(c);
    GH_CUDA(cudaStreamSynchronize(c->stream));
    for (auto& p : c->pending) {
      float ms = 0.f;
      GH_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
      auto it = std::find_if(c->times.begin(), c->times.end(),
                             [&](const auto& kv) { return kv.first == p.name; });
      if (it == c->times.end()) {
        c->times.push_back({p.name, gh::KernelTimes{}});
        it = c->times.end() - 1;
      }
      it->second.ms += ms;
      it->second.count += 1;
      c->event_pool.push_back(p.a);
      c->event_pool.push_back(p.b);
    }
    c->pending.clear();
    double ms = 0.0;
    int64_t n = 0;
    for (const auto& kv : c->times)
      if (kv.first == name) {
        ms = kv.second.ms;
        n = kv.second.count;
      }
    if (total_ms) *total_ms = ms;
    if (count) *count = n;
  });
}

int gh_ctx_reset_timing(gh_ctx* ctx) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c) fail(GH_EINVAL, "ctx: null argument");
    use_device(c);
    GH_CUDA(cudaStreamSynchronize(c->stream));
    for (auto& p : c->pending) {
      c->event_pool.push_back(p.a);
      c->event_pool.push_back(p.b);
    }
    c->pending.clear();
    c->times.clear();
  });
}

int gh_table_build(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid, int32_t scheme,
                   int32_t wrap, gh_table** out) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || !out) fail(GH_EINVAL, "hop table: null argument");
    use_device(c);
    gh::Table* t = new_table(c, wave, grid, scheme);
    try {
      t->wrap = wrap ? 1 : 0;
      gh::build_table_device(c, t, wrap);
      gh::build_plan(c, t);
    } catch (...) {
      free_table(t);
      throw;
    }
    *out = reinterpret_cast<gh_table*>(t);
  });
}

int gh_table_build_shard(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid, int32_t scheme,
                         int32_t wrap, int32_t layer_lo, int32_t layer_hi, gh_table** out) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || !out) fail(GH_EINVAL, "hop table: null argument");
    use_device(c);
    gh::Table* t = new_table(c, wave, grid, scheme);
    const int axis_len = t->slab_hi;
    if (layer_lo < 0 || layer_hi > axis_len || layer_lo >= layer_hi) {
      free_table(t);
      fail(GH_EINVAL, "hop table: shard layers outside the grid");
    }
    const int64_t layer = (int64_t)grid->n[0] * (grid->n[2] > 1 ? grid->n[1] : 1);
    t->slab_lo = layer_lo;
    t->slab_hi = layer_hi;
    t->bin0 = layer_lo * layer;
    t->G = (int64_t)(layer_hi - layer_lo) * layer;
    try {
      t->wrap = wrap ? 1 : 0;
      gh::build_table_device(c, t, wrap);
      gh::build_plan(c, t);
    } catch (...) {
      free_table(t);
      throw;
    }
    *out = reinterpret_cast<gh_table*>(t);
  });
}

int gh_table_set_core(gh_table* table, int32_t core_lo, int32_t core_hi) {
  return guarded([&] {
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!t) fail(GH_EINVAL, "hop table: null argument");
    if (core_lo < t->slab_lo || core_hi > t->slab_hi || core_lo >= core_hi)
      fail(GH_EINVAL, "hop table: core layers outside the shard");
    t->core_lo = core_lo;
    t->core_hi = core_hi;
  });
}

int gh_table_upload(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid, int32_t scheme,
                    const uint32_t* idx, const double* coef, gh_table** out) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || !out || !idx) fail(GH_EINVAL, "hop table: null argument");
    use_device(c);
    gh::Table* t = new_table(c, wave, grid, scheme);
    try {
      const int64_t n = t->G * t->P * t->K;
      for (int64_t i = 0; i < n; ++i)
        if (idx[i] >= static_cast<uint32_t>(t->M))
          fail(GH_ERUNTIME, "hop table: index " + std::to_string(idx[i]) + " outside the FFT grid");
      std::vector<double2> cf(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i)
        cf[static_cast<size_t>(i)] = coef ? make_double2(coef[2 * i], coef[2 * i + 1])
                                          : make_double2(1.0, 0.0);
      GH_CUDA(cudaMalloc(&t->idx_d, sizeof(uint32_t) * n));
      GH_CUDA(cudaMalloc(&t->coef_d, sizeof(double2) * n));
      GH_CUDA(cudaMemcpy(t->idx_d, idx, sizeof(uint32_t) * n, cudaMemcpyHostToDevice));
      GH_CUDA(cudaMemcpy(t->coef_d, cf.data(), sizeof(double2) * n, cudaMemcpyHostToDevice));
      gh::build_plan(c, t);
    } catch (...) {
      free_table(t);
      throw;
    }
    *out = reinterpret_cast<gh_table*>(t);
  });
}

int gh_table_info(const gh_table* table, int64_t* n_bins, int32_t* n_pairs, int32_t* k,
                  int32_t* n_fft, double* max_residual) {
  return guarded([&] {
    auto* t = reinterpret_cast<const gh::Table*>(table);
    if (!t) fail(GH_EINVAL, "hop table: null argument");
    if (n_bins) *n_bins = t->G;
    if (n_pairs) *n_pairs = t->P;
    if (k) *k = t->K;
    if (n_fft) *n_fft = t->M;
    if (max_residual) *max_residual = t->max_residual;
  });
}

int gh_table_download(gh_table* table, uint32_t* idx, double* coef) {
  return guarded([&] {
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!t) fail(GH_EINVAL, "hop table: null argument");
    use_device(t->ctx);
    const int64_t n = t->G * t->P * t->K;
    if (idx) GH_CUDA(cudaMemcpy(idx, t->idx_d, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
    if (coef && t->coef_d) {
      GH_CUDA(cudaMemcpy(coef, t->coef_d, sizeof(double2) * n, cudaMemcpyDeviceToHost));
    } else if (coef) {
      for (int64_t i = 0; i < n; ++i) {  // nearest: unit coefficients (interp.cpp:92)
        coef[2 * i] = 1.0;
        coef[2 * i + 1] = 0.0;
      }
    }
  });
}

// rows of a subset of (global) bins: idx [n][P][K], coef [n][P][K] (re, im)
__global__ void k_table_rows(const uint32_t* idx_d, const double2* coef_d, const int64_t* bins,
                             int64_t n, int64_t bin0, int PK, uint32_t* idx_o, double2* coef_o) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * PK;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / PK, e = i - r * PK;
    const int64_t src = (bins[r] - bin0) * PK + e;
    idx_o[i] = idx_d[src];
    coef_o[i] = coef_d ? coef_d[src] : make_double2(1.0, 0.0);  // nearest: unit (interp.cpp:92)
  }
}

int gh_table_rows(gh_table* table, const int64_t* bins, int64_t n, uint32_t* idx, double* coef) {
  return guarded([&] {
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!t || (n > 0 && (!bins || !idx || !coef))) fail(GH_EINVAL, "hop table: null argument");
    if (n < 0) fail(GH_EINVAL, "hop table: negative row count");
    for (int64_t i = 0; i < n; ++i)
      if (bins[i] < t->bin0 || bins[i] >= t->bin0 + t->G) fail(GH_EINVAL, "hop table: bin out of range");
    if (n == 0) return;
    gh::Ctx* c = t->ctx;
    use_device(c);
    const int PK = t->P * t->K;
    gh::Buffer buf;
    auto* base = static_cast<unsigned char*>(
        buf.get(sizeof(double2) * n * PK + sizeof(int64_t) * n + sizeof(uint32_t) * n * PK));
    auto* co = reinterpret_cast<double2*>(base);
    auto* bd = reinterpret_cast<int64_t*>(base + sizeof(double2) * n * PK);
    auto* io = reinterpret_cast<uint32_t*>(base + sizeof(double2) * n * PK + sizeof(int64_t) * n);
    GH_CUDA(cudaMemcpyAsync(bd, bins, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->stream));
    k_table_rows<<<grid_blocks(n * PK), 256, 0, c->stream>>>(t->idx_d, t->coef_d, bd, n, t->bin0, PK,
                                                             io, co);
    GH_LAUNCHED(c);
    GH_CUDA(cudaMemcpyAsync(idx, io, sizeof(uint32_t) * n * PK, cudaMemcpyDeviceToHost, c->stream));
    GH_CUDA(cudaMemcpyAsync(coef, co, sizeof(double2) * n * PK, cudaMemcpyDeviceToHost, c->stream));
    GH_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int gh_table_destroy(gh_table* table) {
  return guarded([&] {
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!t) return;
    use_device(t->ctx);
    cudaStreamSynchronize(t->ctx->stream);
    free_table(t);
  });
}

int gh_synth_d(gh_ctx* ctx, const gh_wave* wave, const gh_campaign* camp, uint64_t trial0,
               int32_t n_trials, int32_t wrap, float* frames_d, double* truth_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && !frames_d)) fail(GH_EINVAL, "synth: null argument");
    check_wave(wave);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    gh::Buffer txrx;
    const double* tr = upload_txrx(c, wave, txrx);
    const gh::SynthParams sp = make_synth(c, tr, wave->range_scale, camp, trial0, wrap);
    gh::launch_synth(c, sp, n_trials, wave->n_pairs, wave->n_samples,
                     reinterpret_cast<float2*>(frames_d), truth_d);
    check_synth_flag(c, sp);
    txrx.release();
  });
}

int gh_spectra_d(gh_ctx* ctx, const float* frames_d, int32_t n_trials, int32_t n_pairs,
                 int32_t n_samples, int32_t os_range, float* spectra_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && (!frames_d || !spectra_d)))
      fail(GH_EINVAL, "spectra: null argument");
    if (os_range < 1) fail(GH_EINVAL, "spectra: oversampling must be >= 1");
    if (n_pairs < 1 || n_samples < 2) fail(GH_EINVAL, "spectra: bad frame shape");
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    gh::launch_fft(c, reinterpret_cast<const float2*>(frames_d), nullptr, n_trials, n_pairs,
                   n_samples, os_range, 16, gh::FFT_NATURAL, spectra_d);
  });
}

int gh_hop_map_d(gh_ctx* ctx, gh_table* table, const float* frames_d, int32_t n_trials,
                 int32_t combine, float* map_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!c || !t || (n_trials > 0 && (!frames_d || !map_d)))
      fail(GH_EINVAL, "hop: null argument");
    check_combine(combine);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    void* spec = gather_spectra(c, t, reinterpret_cast<const float2*>(frames_d), nullptr,
                                n_trials, combine, true);
    gh::launch_gather(c, t, spec, n_trials, combine, map_d, nullptr);
  });
}

int gh_hop_argmax_d(gh_ctx* ctx, gh_table* table, const float* frames_d, int32_t n_trials,
                    int32_t combine, int64_t* idx_d, float* val_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!c || !t || (n_trials > 0 && (!frames_d || !idx_d || !val_d)))
      fail(GH_EINVAL, "hop: null argument");
    check_combine(combine);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    hop_argmax(c, t, reinterpret_cast<const float2*>(frames_d), nullptr, n_trials, combine, idx_d,
               val_d);
  });
}

int gh_hop_estimate(gh_ctx* ctx, gh_table* table, const double* frames, int32_t n_trials,
                    int32_t combine, int64_t* idx, double* val) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!c || !t || (n_trials > 0 && (!frames || !idx || !val)))
      fail(GH_EINVAL, "hop: null argument");
    check_combine(combine);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    host_frames_pipeline(c, t, frames, n_trials, 1, idx, val,
                         [&](const float2* d64, int tc, int64_t* di, float* dv) {
                           hop_argmax(c, t, d64, nullptr, tc, combine, di, dv);
                         });
  });
}

int gh_hop_estimate_topk(gh_ctx* ctx, gh_table* table, const double* frames, int32_t n_trials,
                         int32_t combine, int32_t k, int64_t* idx, double* val) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!c || !t || (n_trials > 0 && (!frames || !idx || !val)))
      fail(GH_EINVAL, "hop: null argument");
    check_combine(combine);
    if (k < 1 || k > 8) fail(GH_EINVAL, "top-k: k must be in [1, 8]");
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    host_frames_pipeline(c, t, frames, n_trials, k, idx, val,
                         [&](const float2* d64, int tc, int64_t* di, float* dv) {
                           hop_topk(c, t, d64, nullptr, tc, combine, k, di, dv);
                         });
  });
}

int gh_campaign_hop_d(gh_ctx* ctx, gh_table* table, const gh_campaign* camp, uint64_t trial0,
                      int32_t n_trials, int32_t combine, int64_t* idx_d, float* val_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!c || !t || (n_trials > 0 && (!idx_d || !val_d)))
      fail(GH_EINVAL, "campaign: null argument");
    check_combine(combine);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    // the table's window policy (wrap = 0: the reference's window check,
    // reported by the next synchronising call)
    const gh::SynthParams sp = make_campaign_synth(c, t, camp, trial0);
    hop_argmax(c, t, nullptr, &sp, n_trials, combine, idx_d, val_d);
  });
}

int gh_hop_topk_d(gh_ctx* ctx, gh_table* table, const float* frames_d, int32_t n_trials,
                  int32_t combine, int32_t k, int64_t* idx_d, float* val_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!c || !t || (n_trials > 0 && (!frames_d || !idx_d || !val_d)))
      fail(GH_EINVAL, "hop: null argument");
    check_combine(combine);
    if (k < 1 || k > 8) fail(GH_EINVAL, "top-k: k must be in [1, 8]");
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    hop_topk(c, t, reinterpret_cast<const float2*>(frames_d), nullptr, n_trials, combine, k, idx_d,
             val_d);
  });
}

int gh_campaign_hop_topk_d(gh_ctx* ctx, gh_table* table, const gh_campaign* camp, uint64_t trial0,
                           int32_t n_trials, int32_t combine, int32_t k, int64_t* idx_d,
                           float* val_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!c || !t || (n_trials > 0 && (!idx_d || !val_d)))
      fail(GH_EINVAL, "campaign: null argument");
    check_combine(combine);
    if (k < 1 || k > 8) fail(GH_EINVAL, "top-k: k must be in [1, 8]");
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    const gh::SynthParams sp = make_campaign_synth(c, t, camp, trial0);
    hop_topk(c, t, nullptr, &sp, n_trials, combine, k, idx_d, val_d);
  });
}

int gh_topk_local_max_d(gh_ctx* ctx, const gh_grid* grid, const float* map_d, int32_t n_trials,
                        int32_t k, int64_t* idx_d, float* val_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && (!map_d || !idx_d || !val_d)))
      fail(GH_EINVAL, "top-k: null argument");
    grid_size(grid);
    if (k < 1 || k > 8) fail(GH_EINVAL, "top-k: k must be in [1, 8]");
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    gh::launch_topk(c, map_d, n_trials, *grid, k, 0, idx_d, val_d);
  });
}

int gh_direct_map_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid, const float* frames_d,
                    int32_t n_trials, int32_t combine, float* map_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && (!frames_d || !map_d)))
      fail(GH_EINVAL, "decision: null argument");
    check_wave(wave);
    grid_size(grid);
    check_combine(combine);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    gh::Buffer txrx;
    const double* tr = upload_txrx(c, wave, txrx);
    gh::direct_map(c, tr, wave, grid, reinterpret_cast<const float2*>(frames_d), n_trials,
                        combine, map_d, nullptr);
    GH_CUDA(cudaStreamSynchronize(c->stream));
    txrx.release();
  });
}

int gh_direct_argmax_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                       const float* frames_d, int32_t n_trials, int32_t combine, int64_t* idx_d,
                       float* val_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && (!frames_d || !idx_d || !val_d)))
      fail(GH_EINVAL, "decision: null argument");
    check_wave(wave);
    grid_size(grid);
    check_combine(combine);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    gh::Buffer txrx;
    const double* tr = upload_txrx(c, wave, txrx);
    auto* keys = static_cast<unsigned long long*>(c->keys.get(sizeof(unsigned long long) * n_trials));
    GH_CUDA(cudaMemsetAsync(keys, 0, sizeof(unsigned long long) * n_trials, c->stream));
    gh::direct_map(c, tr, wave, grid, reinterpret_cast<const float2*>(frames_d), n_trials,
                        combine, nullptr, keys);
    gh::launch_decode_keys(c, keys, n_trials, idx_d, val_d);
    GH_CUDA(cudaStreamSynchronize(c->stream));
    txrx.release();
  });
}

uint64_t gh_scene_hash(int32_t n_rx, int32_t n_chirps, int32_t n_samples, double f0,
                       double bandwidth, double chirp_duration, const double* tx_xy,
                       const double* rx_xy) {
  Fnv1a f;
  f.u32(static_cast<uint32_t>(n_rx));
  f.u32(static_cast<uint32_t>(n_chirps));
  f.u32(static_cast<uint32_t>(n_samples));
  f.f64(f0);
  f.f64(bandwidth);
  f.f64(chirp_duration);
  f.f64(tx_xy ? tx_xy[0] : 0.0);
  f.f64(tx_xy ? tx_xy[1] : 0.0);
  for (int q = 0; q < n_rx && rx_xy; ++q) {
    f.f64(rx_xy[2 * q]);
    f.f64(rx_xy[2 * q + 1]);
  }
  return f.h;
}

int gh_ght1_write(const char* path, const gh_ght1_header* hdr, const uint32_t* idx,
                  const double* coef) {
  return guarded([&] {
    if (!path || !hdr || !idx) fail(GH_EINVAL, "hop table: null argument");
    ght1_write(path, *hdr, idx, coef);
  });
}

int gh_ght1_read(const char* path, gh_ght1_header* hdr, uint32_t* idx, double* coef,
                 int64_t capacity) {
  return guarded([&] {
    if (!path || !hdr) fail(GH_EINVAL, "hop table: null argument");
    ght1_read(path, *hdr, idx, coef, capacity);
  });
}

int gh_table_save(gh_table* table, const char* path, uint64_t scene_hash) {
  return guarded([&] {
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!t || !path) fail(GH_EINVAL, "hop table: null argument");
    if (t->bin0 != 0 || t->G != (int64_t)t->grid.n[0] * t->grid.n[1] * t->grid.n[2])
      fail(GH_EINVAL, "hop table: a grid shard cannot be saved as GHT1");
    if (t->G > 0xffffffffll) fail(GH_EINVAL, "hop table: too many bins for GHT1");
    const int64_t n = t->G * t->P * t->K;
    std::vector<uint32_t> idx(static_cast<size_t>(n));
    std::vector<double> coef(static_cast<size_t>(2 * n));
    const int st = gh_table_download(table, idx.data(), coef.data());
    if (st != GH_OK) fail(st, g_err);
    gh_ght1_header h{};
    h.n_pairs = t->P;
    h.n_bins = static_cast<int32_t>(t->G);
    h.k = t->K;
    h.os_range = t->os;
    h.n_samples = t->N;
    h.scene_hash = scene_hash;
    h.max_residual = t->max_residual;
    ght1_write(path, h, idx.data(), coef.data());
  });
}

int gh_table_load(gh_ctx* ctx, const char* path, const gh_wave* wave, const gh_grid* grid,
                  uint64_t scene_hash, gh_table** out) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || !path || !out) fail(GH_EINVAL, "hop table: null argument");
    check_wave(wave);
    const int64_t G = grid_size(grid);
    gh_ght1_header h{};
    ght1_read(path, h, nullptr, nullptr, 0);
    // bind to the scene and grid this table is about to serve
    // (interp.cpp:382-386; os_range too, since the spectra follow the wave)
    if (h.scene_hash != scene_hash || h.n_pairs != wave->n_pairs ||
        h.n_samples != wave->n_samples || h.os_range != wave->os_range || (int64_t)h.n_bins != G)
      fail(GH_ERUNTIME, std::string(path) + ": stale hop table (scene or grid mismatch)");
    const int64_t n = G * h.n_pairs * h.k;
    std::vector<uint32_t> idx(static_cast<size_t>(n));
    std::vector<double> coef(static_cast<size_t>(2 * n));
    ght1_read(path, h, idx.data(), coef.data(), n);
    gh_table* t = nullptr;
    const int st = gh_table_upload(ctx, wave, grid, h.k, idx.data(), coef.data(), &t);
    if (st != GH_OK) fail(st, g_err);
    reinterpret_cast<gh::Table*>(t)->max_residual = h.max_residual;
    *out = t;
  });
}

int gh_multilaterate_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                       const double* rhat_d, int32_t n_trials, int64_t* idx_d, double* res_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && (!rhat_d || !idx_d || !res_d)))
      fail(GH_EINVAL, "multilateration: null argument");
    check_wave(wave);
    grid_size(grid);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    gh::Buffer txrx;
    const double* tr = upload_txrx(c, wave, txrx);
    gh::launch_multilaterate(c, tr, wave, grid, rhat_d, n_trials, idx_d, res_d);
    GH_CUDA(cudaStreamSynchronize(c->stream));
    txrx.release();
  });
}

int gh_indirect_argmin_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                         const float* frames_d, int32_t n_trials, double* rhat_d, int64_t* idx_d,
                         double* res_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && (!frames_d || !idx_d || !res_d)))
      fail(GH_EINVAL, "indirect: null argument");
    check_wave(wave);
    grid_size(grid);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    const int P = wave->n_pairs, N = wave->n_samples, M = N * wave->os_range;
    const int64_t rows = (int64_t)n_trials * P;
    // natural complex spectra [T][P][M], then r_hat [T][P] (caller's or scratch)
    const size_t spec_bytes = sizeof(float2) * rows * M;
    auto* base = static_cast<unsigned char*>(
        c->spectra.get(spec_bytes + (rhat_d ? 0 : sizeof(double) * rows)));
    auto* spec = reinterpret_cast<float2*>(base);
    double* rh = rhat_d ? rhat_d : reinterpret_cast<double*>(base + spec_bytes);
    gh::launch_fft(c, reinterpret_cast<const float2*>(frames_d), nullptr, n_trials, P, N,
                   wave->os_range, 16, gh::FFT_NATURAL, spec);
    gh::launch_range_peaks(c, spec, rows, M, wave->os_range, rh);
    gh::Buffer txrx;
    const double* tr = upload_txrx(c, wave, txrx);
    gh::launch_multilaterate(c, tr, wave, grid, rh, n_trials, idx_d, res_d);
    GH_CUDA(cudaStreamSynchronize(c->stream));
    txrx.release();
  });
}

int gh_hop_map_mc_d(gh_ctx* ctx, gh_table* table, const float* frames_d, int32_t n_trials,
                    int32_t n_chirps, float* map_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!c || !t || (n_trials > 0 && (!frames_d || !map_d))) fail(GH_EINVAL, "hop: null argument");
    if (n_chirps < 1) fail(GH_EINVAL, "waveform: n_chirps must be >= 1");
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    hop_mc(c, t, reinterpret_cast<const float2*>(frames_d), n_trials, n_chirps, map_d, nullptr,
           nullptr);
    GH_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int gh_hop_argmax_mc_d(gh_ctx* ctx, gh_table* table, const float* frames_d, int32_t n_trials,
                       int32_t n_chirps, int64_t* idx_d, float* val_d) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!c || !t || (n_trials > 0 && (!frames_d || !idx_d || !val_d)))
      fail(GH_EINVAL, "hop: null argument");
    if (n_chirps < 1) fail(GH_EINVAL, "waveform: n_chirps must be >= 1");
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    hop_mc(c, t, reinterpret_cast<const float2*>(frames_d), n_trials, n_chirps, nullptr, idx_d,
           val_d);
    GH_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int gh_mrf1_write(const char* path, const gh_mrf1_header* hdr, const double* rx_xy,
                  const double* frames) {
  return guarded([&] {
    if (!path || !hdr || !rx_xy || (hdr->n_frames > 0 && !frames))
      fail(GH_EINVAL, "capture: null argument");
    if (hdr->n_frames < 0) fail(GH_EINVAL, "capture: frame count must be >= 0");
    mrf1_validate(*hdr, rx_xy);
    const size_t samples = (size_t)hdr->n_frames * hdr->n_rx * hdr->n_chirps * hdr->n_samples;
    std::string out;
    out.reserve(24 + 24 + (size_t)(hdr->n_rx + 1) * 16 + samples * 16);
    out.append("MRF1", 4);
    ght1_put<uint32_t>(out, kMrf1Version);
    ght1_put<uint32_t>(out, (uint32_t)hdr->n_rx);
    ght1_put<uint32_t>(out, (uint32_t)hdr->n_chirps);
    ght1_put<uint32_t>(out, (uint32_t)hdr->n_samples);
    ght1_put<uint32_t>(out, (uint32_t)hdr->n_frames);
    ght1_put<double>(out, hdr->f0);
    ght1_put<double>(out, hdr->bandwidth);
    ght1_put<double>(out, hdr->chirp_duration);
    ght1_put<double>(out, hdr->tx[0]);
    ght1_put<double>(out, hdr->tx[1]);
    for (int q = 0; q < hdr->n_rx; ++q) {
      ght1_put<double>(out, rx_xy[2 * q]);
      ght1_put<double>(out, rx_xy[2 * q + 1]);
    }
    // frames receiver-major, each matrix row-major: exactly [T][Q][Mc][Ms]
    out.append(reinterpret_cast<const char*>(frames), samples * 16);
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) fail(GH_ERUNTIME, std::string(path) + ": cannot open for writing");
    f.write(out.data(), static_cast<std::streamsize>(out.size()));
    f.flush();
    if (!f) fail(GH_ERUNTIME, std::string(path) + ": short write");
  });
}

int gh_mrf1_read(const char* path, gh_mrf1_header* hdr, double* rx_xy, int32_t rx_capacity,
                 double* frames, int64_t capacity) {
  return guarded([&] {
    if (!path || !hdr) fail(GH_EINVAL, "capture: null argument");
    const std::string p(path);
    const std::string data = ght1_read_file(p);
    Ght1Reader rd{data.data(), data.size(), p};
    rd.need(4, "magic");
    if (std::memcmp(rd.p, "MRF1", 4) != 0)
      fail(GH_ERUNTIME, p + ": bad magic (not an MRF1 capture)");
    rd.p += 4;
    rd.left -= 4;
    const uint32_t version = rd.get<uint32_t>("version");
    if (version != kMrf1Version)
      fail(GH_ERUNTIME, p + ": unsupported capture version " + std::to_string(version));
    gh_mrf1_header h{};
    h.n_rx = (int32_t)rd.get<uint32_t>("receiver count");
    h.n_chirps = (int32_t)rd.get<uint32_t>("chirp count");
    h.n_samples = (int32_t)rd.get<uint32_t>("sample count");
    h.n_frames = (int32_t)rd.get<uint32_t>("frame count");
    h.f0 = rd.get<double>("carrier");
    h.bandwidth = rd.get<double>("bandwidth");
    h.chirp_duration = rd.get<double>("chirp duration");
    h.tx[0] = rd.get<double>("TX coordinate");
    h.tx[1] = rd.get<double>("TX coordinate");
    std::vector<double> rx(2 * (size_t)(uint32_t)h.n_rx);
    for (size_t q = 0; q < rx.size(); ++q) rx[q] = rd.get<double>("RX coordinate");
    mrf1_validate(h, rx.data());
    const size_t samples = (size_t)(uint32_t)h.n_frames * (uint32_t)h.n_rx * (uint32_t)h.n_chirps *
                           (uint32_t)h.n_samples;
    if (rd.left != samples * 16)
      fail(GH_ERUNTIME, p + ": payload size mismatch (expected " + std::to_string(samples * 16) +
                            " bytes, have " + std::to_string(rd.left) + ")");
    *hdr = h;
    if (rx_xy) {
      if (rx_capacity < h.n_rx) fail(GH_EINVAL, "capture: receiver array too small");
      std::memcpy(rx_xy, rx.data(), sizeof(double) * rx.size());
    }
    if (frames) {
      if (capacity < (int64_t)samples) fail(GH_EINVAL, "capture: frame array too small");
      std::memcpy(frames, rd.p, samples * 16);
    }
  });
}

static int velocity_entry(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                          const gh_velocity_grid* vg, const float* frames_d, int32_t n_trials,
                          int32_t n_chirps, const int64_t* loc_d, int64_t* vidx_d, float* vval_d,
                          bool hop) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || !vg || (n_trials > 0 && (!frames_d || !loc_d || !vidx_d || !vval_d)))
      fail(GH_EINVAL, "velocity: null argument");
    check_wave(wave);
    grid_size(grid);
    if (n_chirps < 1) fail(GH_EINVAL, "waveform: n_chirps must be >= 1");
    if (vg->half < 0) fail(GH_EINVAL, hop ? "hop velocity: empty grid" : "velocity scan: empty grid");
    if (hop && vg->os_doppler < 1) fail(GH_EINVAL, "hop velocity: oversampling must be >= 1");
    if (!(std::isfinite(vg->doppler_scale) && std::isfinite(vg->spacing) && vg->spacing > 0.0))
      fail(GH_EINVAL, "velocity grid: spacing must be positive");
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    gh::Buffer txrx;
    const double* tr = upload_txrx(c, wave, txrx);
    gh::launch_velocity(c, tr, wave, grid, vg, reinterpret_cast<const float2*>(frames_d),
                        n_trials, n_chirps, loc_d, hop, vidx_d, vval_d);
    GH_CUDA(cudaStreamSynchronize(c->stream));
    txrx.release();
  });
}

int gh_hop_velocity_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                      const gh_velocity_grid* vgrid, const float* frames_d, int32_t n_trials,
                      int32_t n_chirps, const int64_t* loc_d, int64_t* vidx_d, float* vval_d) {
  return velocity_entry(ctx, wave, grid, vgrid, frames_d, n_trials, n_chirps, loc_d, vidx_d,
                        vval_d, true);
}

int gh_direct_velocity_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                         const gh_velocity_grid* vgrid, const float* frames_d,
                         int32_t n_trials, int32_t n_chirps, const int64_t* loc_d,
                         int64_t* vidx_d, float* vval_d) {
  return velocity_entry(ctx, wave, grid, vgrid, frames_d, n_trials, n_chirps, loc_d, vidx_d,
                        vval_d, false);
}

}  // extern "C"

extern "C" {

int gh_comm_unique_id(uint8_t id[GH_COMM_ID_BYTES]) {
  return guarded([&] {
    if (!id) fail(GH_EINVAL, "comm: null argument");
    gh::comm_unique_id(id);
  });
}

int gh_comm_init(gh_ctx* ctx, const uint8_t id[GH_COMM_ID_BYTES], int32_t n_ranks, int32_t rank,
                 gh_comm** out) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || !id || !out) fail(GH_EINVAL, "comm: null argument");
    use_device(c);
    *out = reinterpret_cast<gh_comm*>(gh::comm_init(c, id, n_ranks, rank));
  });
}

int gh_comm_info(const gh_comm* comm, int32_t* n_ranks, int32_t* rank) {
  return guarded([&] {
    if (!comm || !n_ranks || !rank) fail(GH_EINVAL, "comm: null argument");
    int n = 0, r = 0;
    gh::comm_info(reinterpret_cast<const gh::Comm*>(comm), &n, &r);
    *n_ranks = n;
    *rank = r;
  });
}

int gh_comm_destroy(gh_comm* comm) {
  return guarded([&] { gh::comm_destroy(reinterpret_cast<gh::Comm*>(comm)); });
}

int gh_campaign_run(gh_ctx* ctx, gh_comm* comm, const gh_campaign_desc* desc, gh_cell_stats* out,
                    int32_t capacity, int32_t* n_cells) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c) fail(GH_EINVAL, "campaign: null argument");
    use_device(c);
    gh::campaign_run(c, reinterpret_cast<gh::Comm*>(comm), desc, out, capacity, n_cells);
  });
}

}  // extern "C"

// ---- host-buffer forms of the stage entry points (the C++ wrappers'
// reference signatures: synth.hpp:26-36, hopping.hpp:14-22, direct.hpp:19-39,
// interp.hpp:41). complex128 in / out as the reference's CMat; the compute
// runs on the device in fp32 (fp64 for the table / fit) as the _d forms.
extern "C" {

int gh_table_geometry(const gh_table* table, int32_t* n_samples, int32_t* os_range,
                      double* range_scale) {
  return guarded([&] {
    auto* t = reinterpret_cast<const gh::Table*>(table);
    if (!t) fail(GH_EINVAL, "hop table: null argument");
    if (n_samples) *n_samples = t->N;
    if (os_range) *os_range = t->os;
    if (range_scale) *range_scale = t->scale;
  });
}

int gh_spectra(gh_ctx* ctx, const double* frames, int32_t n_trials, int32_t n_pairs,
               int32_t n_samples, int32_t os_range, double* spectra) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && (!frames || !spectra))) fail(GH_EINVAL, "spectra: null argument");
    if (os_range < 1) fail(GH_EINVAL, "spectra: oversampling must be >= 1");
    if (n_pairs < 1 || n_samples < 2 || n_trials < 0) fail(GH_EINVAL, "spectra: bad frame shape");
    if (n_trials == 0) return;
    use_device(c);
    gh::Buffer in, out;
    const int64_t rows = (int64_t)n_trials * n_pairs, M = (int64_t)n_samples * os_range;
    const float2* f = frames_to_device(c, in, frames, rows * n_samples);
    auto* base = static_cast<unsigned char*>(out.get((sizeof(float2) + sizeof(double2)) * rows * M));
    auto* s64 = reinterpret_cast<float2*>(base);
    auto* s128 = reinterpret_cast<double2*>(base + sizeof(float2) * rows * M);
    gh::launch_fft(c, f, nullptr, n_trials, n_pairs, n_samples, os_range, 16, gh::FFT_NATURAL, s64);
    k_c64_to_c128<<<grid_blocks(rows * M), 256, 0, c->stream>>>(s64, s128, rows * M);
    GH_LAUNCHED(c);
    GH_CUDA(cudaMemcpyAsync(spectra, s128, sizeof(double2) * rows * M, cudaMemcpyDeviceToHost,
                            c->stream));
    GH_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int gh_hop_map(gh_ctx* ctx, gh_table* table, const double* frames, int32_t n_trials,
               int32_t combine, double* map) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    auto* t = reinterpret_cast<gh::Table*>(table);
    if (!c || !t || (n_trials > 0 && (!frames || !map))) fail(GH_EINVAL, "hop: null argument");
    check_combine(combine);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    gh::Buffer in, m32, m64;
    const float2* f = frames_to_device(c, in, frames, (int64_t)n_trials * t->P * t->N);
    auto* m = static_cast<float*>(m32.get(sizeof(float) * n_trials * t->G));
    void* spec = gather_spectra(c, t, f, nullptr, n_trials, combine, true);
    gh::launch_gather(c, t, spec, n_trials, combine, m, nullptr);
    values_to_host(c, m64, m, (int64_t)n_trials * t->G, map);
  });
}

int gh_direct_map(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid, const double* frames,
                  int32_t n_trials, int32_t combine, double* map) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && (!frames || !map))) fail(GH_EINVAL, "decision: null argument");
    check_wave(wave);
    const int64_t G = grid_size(grid);
    check_combine(combine);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    gh::Buffer in, txrx, m32, m64;
    const float2* f = frames_to_device(c, in, frames, (int64_t)n_trials * wave->n_pairs * wave->n_samples);
    const double* tr = upload_txrx(c, wave, txrx);
    auto* m = static_cast<float*>(m32.get(sizeof(float) * n_trials * G));
    gh::direct_map(c, tr, wave, grid, f, n_trials, combine, m, nullptr);
    values_to_host(c, m64, m, (int64_t)n_trials * G, map);
  });
}

int gh_direct_estimate(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid, const double* frames,
                       int32_t n_trials, int32_t combine, int64_t* idx, double* val) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && (!frames || !idx || !val))) fail(GH_EINVAL, "decision: null argument");
    check_wave(wave);
    grid_size(grid);
    check_combine(combine);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    gh::Buffer in, txrx, res, v64;
    const float2* f = frames_to_device(c, in, frames, (int64_t)n_trials * wave->n_pairs * wave->n_samples);
    const double* tr = upload_txrx(c, wave, txrx);
    auto* base = static_cast<unsigned char*>(
        res.get((sizeof(unsigned long long) + sizeof(int64_t) + sizeof(float)) * n_trials));
    auto* keys = reinterpret_cast<unsigned long long*>(base);
    auto* di = reinterpret_cast<int64_t*>(keys + n_trials);
    auto* dv = reinterpret_cast<float*>(di + n_trials);
    GH_CUDA(cudaMemsetAsync(keys, 0, sizeof(unsigned long long) * n_trials, c->stream));
    gh::direct_map(c, tr, wave, grid, f, n_trials, combine, nullptr, keys);
    gh::launch_decode_keys(c, keys, n_trials, di, dv);
    GH_CUDA(cudaMemcpyAsync(idx, di, sizeof(int64_t) * n_trials, cudaMemcpyDeviceToHost, c->stream));
    values_to_host(c, v64, dv, n_trials, val);
  });
}

int gh_synth(gh_ctx* ctx, const gh_wave* wave, const gh_campaign* camp, uint64_t trial0,
             int32_t n_trials, int32_t wrap, double* frames, double* truth) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && !frames)) fail(GH_EINVAL, "synth: null argument");
    check_wave(wave);
    if (n_trials < 0) fail(GH_EINVAL, "trials must be >= 0");
    if (n_trials == 0) return;
    use_device(c);
    gh::Buffer txrx, buf;
    const int64_t n = (int64_t)n_trials * wave->n_pairs * wave->n_samples;
    const int64_t nt = (int64_t)n_trials * camp->n_targets * 3;
    auto* base = static_cast<unsigned char*>(
        buf.get(sizeof(float2) * n + sizeof(double2) * n + sizeof(double) * nt));
    auto* f64 = reinterpret_cast<float2*>(base);
    auto* f128 = reinterpret_cast<double2*>(base + sizeof(float2) * n);
    auto* tr_d = reinterpret_cast<double*>(base + sizeof(float2) * n + sizeof(double2) * n);
    const double* tr = upload_txrx(c, wave, txrx);
    const gh::SynthParams sp = make_synth(c, tr, wave->range_scale, camp, trial0, wrap);
    gh::launch_synth(c, sp, n_trials, wave->n_pairs, wave->n_samples, f64, tr_d);
    check_synth_flag(c, sp);
    k_c64_to_c128<<<grid_blocks(n), 256, 0, c->stream>>>(f64, f128, n);
    GH_LAUNCHED(c);
    GH_CUDA(cudaMemcpyAsync(frames, f128, sizeof(double2) * n, cudaMemcpyDeviceToHost, c->stream));
    if (truth)
      GH_CUDA(cudaMemcpyAsync(truth, tr_d, sizeof(double) * nt, cudaMemcpyDeviceToHost, c->stream));
    GH_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int gh_add_noise(gh_ctx* ctx, double* frames, int32_t n_trials, int32_t n_pairs, int32_t n_samples,
                 uint64_t seed, uint64_t trial0, double snr_db) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n_trials > 0 && !frames)) fail(GH_EINVAL, "noise: null argument");
    if (n_trials < 0 || n_pairs < 1 || n_samples < 1) fail(GH_EINVAL, "noise: bad frame shape");
    if (!std::isfinite(snr_db)) return;  // NoiseSpec without SNR: noiseless (synth.cpp:41)
    if (n_trials == 0) return;
    use_device(c);
    gh::Buffer buf;
    const int64_t n = (int64_t)n_trials * n_pairs * n_samples;
    auto* d = static_cast<double2*>(buf.get(sizeof(double2) * n));
    GH_CUDA(cudaMemcpyAsync(d, frames, sizeof(double2) * n, cudaMemcpyHostToDevice, c->stream));
    gh::launch_add_noise(c, d, n_trials, n_pairs, n_samples, seed, trial0,
                         std::pow(10.0, -snr_db / 20.0));
    GH_CUDA(cudaMemcpyAsync(frames, d, sizeof(double2) * n, cudaMemcpyDeviceToHost, c->stream));
    GH_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int gh_fit_atom(gh_ctx* ctx, int32_t n_samples, int32_t os_range, const double* r, int32_t n,
                int32_t scheme, uint32_t* idx, double* coef, double* residual) {
  return guarded([&] {
    auto* c = reinterpret_cast<gh::Ctx*>(ctx);
    if (!c || (n > 0 && (!r || !idx || !coef || !residual))) fail(GH_EINVAL, "fit: null argument");
    if (n_samples < 2) fail(GH_EINVAL, "waveform: n_samples must be >= 2");
    if (os_range < 1) fail(GH_EINVAL, "hop table: oversampling must be >= 1");
    if (scheme < GH_NEAREST || scheme > GH_POLAR) fail(GH_EINVAL, "unknown interpolation scheme");
    for (int32_t i = 0; i < n; ++i)
      if (!std::isfinite(r[i])) fail(GH_EINVAL, "fit_atom: range must be finite");
    if (n <= 0) return;
    use_device(c);
    gh::Buffer buf;
    auto* base = static_cast<unsigned char*>(
        buf.get(sizeof(double) * n + sizeof(uint32_t) * 3 * n + sizeof(double2) * 3 * n + sizeof(double) * n));
    // double2 first: every sub-array stays aligned for any n
    auto* cd = reinterpret_cast<double2*>(base);
    auto* rd = reinterpret_cast<double*>(base + sizeof(double2) * 3 * n);
    auto* res = reinterpret_cast<double*>(base + sizeof(double2) * 3 * n + sizeof(double) * n);
    auto* id = reinterpret_cast<uint32_t*>(base + sizeof(double2) * 3 * n + 2 * sizeof(double) * n);
    GH_CUDA(cudaMemcpyAsync(rd, r, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    gh::launch_fit_atoms(c, n_samples, os_range, rd, n, scheme, id, cd, res);
    GH_CUDA(cudaMemcpyAsync(idx, id, sizeof(uint32_t) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
    GH_CUDA(cudaMemcpyAsync(coef, cd, sizeof(double2) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
    GH_CUDA(cudaMemcpyAsync(residual, res, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    GH_CUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
