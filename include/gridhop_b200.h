/*
 * gridhop_b200.h — C ABI of the B200-native grid-hopping hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch or CUDA
 * types, no exceptions across the ABI. Every call returns an int status and
 * leaves a thread-local message readable through gh_last_error(). Status
 * codes map 1:1 onto the exception types of the reference library
 * (/root/reference/proj/core), so the C++ wrappers in gridhop_b200.hpp can
 * rethrow exactly what the reference throws:
 *
 *   GH_OK        0   success
 *   GH_EINVAL    1   std::invalid_argument   (bad sizes / arguments)
 *   GH_ERUNTIME  2   std::runtime_error      (stale table, window errors)
 *   GH_EDOMAIN   3   std::domain_error       (degenerate geometry)
 *   GH_ECUDA     4   std::runtime_error      (CUDA / device failure)
 *
 * Suffix `_d`: every array argument is a DEVICE pointer on the context's
 * device (e.g. torch.Tensor.data_ptr()). No suffix: HOST pointers; the call
 * does its own host<->device copies on the context stream and returns when
 * the results are in host memory.
 *
 * Which reference interface each entry point replaces is given beside it
 * (file:line under /root/reference/proj/core). The reference binds none of
 * these today (it has no FFI); INTEGRATION.md shows the C++ wrapper and
 * ctypes bindings a maintainer would add.
 */
#ifndef GRIDHOP_B200_H
#define GRIDHOP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GH_ABI_VERSION 1

enum gh_status { GH_OK = 0, GH_EINVAL = 1, GH_ERUNTIME = 2, GH_EDOMAIN = 3, GH_ECUDA = 4 };

/* InterpScheme (include/gridhop/interp.hpp:16) + the polar scheme. */
enum gh_scheme { GH_NEAREST = 1, GH_LINEAR = 2, GH_POLY3 = 3, GH_POLAR = 4 };

/* Non-coherent combine over pairs: power sum |.|^2 (the reference,
 * src/hopping.cpp:99) or magnitude sum |.| (BASELINE c1 wording). */
enum gh_combine { GH_POWER = 0, GH_MAGNITUDE = 1 };

/* Waveform + TX/RX pair list. Generalises WaveformConfig + SceneGeometry
 * (include/gridhop/model.hpp:21-50) to P (tx, rx) pairs in 3-D. */
typedef struct {
  int32_t n_samples;   /* N fast-time samples per pair                    */
  int32_t os_range;    /* zero-padding factor; M = os_range * N           */
  double range_scale;  /* B / c: fast-time bins per metre of summed path  */
  int32_t n_pairs;     /* P                                               */
  const double* tx;    /* host [P][3] TX positions, metres                */
  const double* rx;    /* host [P][3] RX positions, metres                */
} gh_wave;

/* LocationGrid (include/gridhop/model.hpp:77-92) in 3-D, x fastest. */
typedef struct {
  double origin[3];
  double spacing[3];
  int32_t n[3];
} gh_grid;

/* Monte-Carlo scene model: sample_scene (src/montecarlo.cpp:48-66) with the
 * BASELINE extensions (K targets, per-pair amplitude / SNR). */
typedef struct {
  uint64_t seed;
  int32_t n_targets;
  int32_t dims;            /* 2 or 3 position draws per target            */
  double area_lo[3];
  double area_hi[3];
  int32_t amp_mode;        /* 0 unit-phase shared, 1 unit-phase per pair,
                              2 CN(0,1) shared, 3 CN(0,1) per pair         */
  int32_t snr_mode;        /* 0 fixed, 1 U[snr_lo, snr_hi] per pair,
                              2 noiseless                                  */
  double snr_db;
  double snr_lo;
  double snr_hi;
} gh_campaign;

typedef struct gh_ctx gh_ctx;      /* one device + one stream + scratch    */
typedef struct gh_table gh_table;  /* device-resident mapping operator     */

/* ---- library / context ------------------------------------------------ */
const char* gh_last_error(void);
int gh_abi_version(void);
int gh_ctx_create(int32_t device, gh_ctx** out);
int gh_ctx_destroy(gh_ctx* ctx);
/* The stream every call of this context is enqueued on (cudaStream_t). */
int gh_ctx_get_stream(gh_ctx* ctx, void** stream);
/* Use a caller-owned stream instead (e.g. torch.cuda.current_stream()). */
int gh_ctx_set_stream(gh_ctx* ctx, void* stream);
int gh_ctx_synchronize(gh_ctx* ctx);
/* Number of kernels this context has launched (bench `gpu_launches`). */
int gh_ctx_launch_count(gh_ctx* ctx, int64_t* count);
/* Per-kernel CUDA-event timing on the context stream (off by default).
 * gh_ctx_kernel_time synchronises, then reports the accumulated device time
 * and launch count of kernels named `name` ("fft", "synth_fft", "gather",
 * "decode", "convert", "direct_simt", "direct_umma", "synth") since the last
 * reset. */
int gh_ctx_set_timing(gh_ctx* ctx, int32_t on);
int gh_ctx_kernel_time(gh_ctx* ctx, const char* name, double* total_ms, int64_t* count);
int gh_ctx_reset_timing(gh_ctx* ctx);
/* Direct-method engine: 0 = tcgen05 tensor cores, 3xFP16 (kind::f16 on
 * power-of-two-scaled frames), warp-specialised pipeline (default); 1 =
 * CUDA-core fp32 contraction (the reference path the tensor-core kernels are
 * checked and timed against); 2 = single-stage tcgen05 3xTF32 kernel (v1);
 * 3 = the warp-specialised pipeline in 3xTF32 (kind::tf32); 4 = the same
 * pipeline with one fp16 MMA per K step (1xFP16 fast mode: a third of the
 * tensor work; fp16 operands leave the c2 maps ~8e-5 of their maximum off,
 * marginal against the 1e-4 parity bar, so it is never the default). */
int gh_ctx_set_direct_impl(gh_ctx* ctx, int32_t impl);
/* Top-K local-maximum engine (BASELINE c3): 0 = auto (engine 3 where the
 * table's plan admits it — tiled K = 1 plans of at most 16 pairs — and the
 * call's 8-trial batches fill its rounds of one batch per SM, else engine 2);
 * 1 = halo tiles with the tile's values in shared memory; 2 = map-mode gather, then
 * k_topk_localmax over the maps in HBM; 3 = the gather with the prune test in
 * its loop and candidates verified against the table and spectra (no maps).
 * All engines return identical bins and values. */
int gh_ctx_set_topk_impl(gh_ctx* ctx, int32_t impl);
/* Debug builds of the hand-rolled pipelines (compute-sanitizer's stand-in):
 * with on != 0, kernels that have a bounds-tested instantiation run it — the
 * top-K pick gather tests every staged shared-memory offset, window extent,
 * candidate-queue slot and table / spectra row it touches — and a violation
 * fails the call with GH_ERUNTIME. Same results, slower, synchronous. */
int gh_ctx_set_debug_checks(gh_ctx* ctx, int32_t on);
/* Diagnostics: measured shared-memory (LSU) read bandwidth of the device,
 * GB/s, all SMs — the roofline denominator of the gather kernel. */
int gh_measure_smem_peak(gh_ctx* ctx, double* gbps);

/* ---- mapping operator (offline) --------------------------------------- */
/* precompute_hop_table (src/interp.cpp:156-223) on the device in fp64.
 * wrap = 0 keeps the reference's window check (GH_ERUNTIME naming the
 * offending bins, interp.cpp:182-201); wrap = 1 relies on the atoms'
 * periodicity (interp.cpp:39-44) for aliasing scenes (BASELINE c1/c2). */
int gh_table_build(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                   int32_t scheme, int32_t wrap, gh_table** out);
/* Location-grid shard (BASELINE c5): the operator for layers
 * [layer_lo, layer_hi) of the grid's z axis (3-D grids) or y axis (2-D) —
 * one contiguous range of global bins. Grid points are computed from the
 * full grid, so rows are bit-identical to the full table's; every bin index
 * this table reports (argmax, top-k) is global, so per-GPU shard winners
 * merge with one all-reduce(max) of the 64-bit key. Maps are shard-local. */
int gh_table_build_shard(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                         int32_t scheme, int32_t wrap, int32_t layer_lo,
                         int32_t layer_hi, gh_table** out);
/* Halo shards for multi-target picks across location-grid shards: a shard
 * built one layer beyond its core on each interior side reports top-k
 * local maxima of the core layers [core_lo, core_hi) only (global layer
 * indices inside the shard); the halo layers complete the neighbourhoods of
 * the core's border bins, so per-shard candidates merge exactly (all-gather
 * of K keys per trial, then the K best). */
int gh_table_set_core(gh_table* table, int32_t core_lo, int32_t core_hi);
/* load_hop_table (src/interp.cpp:318-389) analogue: host arrays in the
 * reference layout [bin][pair][K] (HopTable::entry_offset, interp.hpp:55-59);
 * coef = complex128 (re, im) pairs, NULL means all ones (K = 1). */
int gh_table_upload(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                    int32_t scheme, const uint32_t* idx, const double* coef,
                    gh_table** out);
int gh_table_info(const gh_table* t, int64_t* n_bins, int32_t* n_pairs,
                  int32_t* k, int32_t* n_fft, double* max_residual);
/* Copy the operator back in the reference layout (host pointers). */
int gh_table_download(gh_table* t, uint32_t* idx, double* coef);
/* Rows of a subset of the table's (global) bins, the layout of
 * gh_table_download: idx [n][P][K], coef [n][P][K] (re, im) — spot checks of
 * tables too large to download (BASELINE c5: 16.7M bins x 64 pairs). */
int gh_table_rows(gh_table* table, const int64_t* bins, int64_t n, uint32_t* idx, double* coef);
int gh_table_destroy(gh_table* t);

/* ---- MRF1 capture container ---------------------------------------------
 * write_frames / read_frames (src/frame_io.cpp:53-164, format
 * include/gridhop/frame_io.hpp:10-16): little-endian "MRF1", u32 version (1)
 * / Q / Mc / Ms / frame count, f64 f0 / bandwidth / chirp duration, (Q+1)
 * coordinate pairs (TX first), then frames receiver-major, each matrix
 * row-major, entries as (re, im) f64 — i.e. complex128 [T][Q][Mc][Ms].
 * Validation errors are GH_EINVAL with the reference's texts ("waveform:
 * n_chirps must be >= 2", ...); file errors GH_ERUNTIME ("<path>: bad magic
 * (not an MRF1 capture)", "<path>: payload size mismatch ...", ...).
 * gh_mrf1_read with rx_xy = frames = NULL reads the header only. */
typedef struct gh_mrf1_header {
  int32_t n_rx;
  int32_t n_chirps;
  int32_t n_samples;
  int32_t n_frames;
  double f0;
  double bandwidth;
  double chirp_duration;
  double tx[2];
} gh_mrf1_header;
int gh_mrf1_write(const char* path, const gh_mrf1_header* hdr, const double* rx_xy,
                  const double* frames);
int gh_mrf1_read(const char* path, gh_mrf1_header* hdr, double* rx_xy, int32_t rx_capacity,
                 double* frames, int64_t capacity);

/* ---- multi-chirp frames (the reference's slow-time axis, Mc > 1) --------
 * scan_planes / hop_bin_value over Mc chirps (src/hopping.cpp:59-117):
 * value(bin) = sum_q sum_mc |Z_q(mc, I(bin, q))|^2 for K = 1 (nearest)
 * tables, power combine. frames complex64 [T][P][Mc][N] (a FrameSet per
 * trial, receiver-major, each matrix row-major); map fp32 [T][G]. */
int gh_hop_map_mc_d(gh_ctx* ctx, gh_table* table, const float* frames_d, int32_t n_trials,
                    int32_t n_chirps, float* map_d);
int gh_hop_argmax_mc_d(gh_ctx* ctx, gh_table* table, const float* frames_d, int32_t n_trials,
                       int32_t n_chirps, int64_t* idx_d, float* val_d);

/* ---- velocity stage at the located bins ----------------------------------
 * hop_velocity (src/hopping.cpp:185-236) and direct_velocity
 * (src/direct.cpp:145-228) for T trials of multi-chirp frames, each at its
 * located bin loc_d[t] (e.g. from gh_hop_argmax_mc_d): range compression at
 * x_hat, then the velocity-grid scan — hop: nearest bins of the zero-padded
 * slow-time spectrum (n_d = os_doppler * Mc; Mc and os_doppler powers of
 * two); direct: exact correlation with each pair's Doppler atom. The grid is
 * VelocityGrid (model.hpp:93-107): point k = spacing * (k % n - half,
 * k / n - half), n = 2 half + 1; first maximum wins. frames complex64
 * [T][P][Mc][N]; out velocity-grid index int64 [T] and value fp32 [T]. */
typedef struct gh_velocity_grid {
  double doppler_scale;  /* WaveformConfig::doppler_scale = f0 Tc Mc / c   */
  double spacing;        /* VelocityGrid::spacing, m/s                     */
  int32_t half;          /* VelocityGrid::half                             */
  int32_t os_doppler;    /* hop: slow-time zero padding (>= 1)             */
} gh_velocity_grid;
int gh_hop_velocity_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                      const gh_velocity_grid* vgrid, const float* frames_d, int32_t n_trials,
                      int32_t n_chirps, const int64_t* loc_d, int64_t* vidx_d, float* vval_d);
int gh_direct_velocity_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                         const gh_velocity_grid* vgrid, const float* frames_d,
                         int32_t n_trials, int32_t n_chirps, const int64_t* loc_d,
                         int64_t* vidx_d, float* vval_d);

/* ---- indirect pipeline, location stage ---------------------------------
 * range_doppler_map + RangeDopplerMap::peak + multilaterate_location
 * (src/indirect.cpp:10-83) at Mc = 1: per (trial, pair) r_hat = (first
 * maximum bin of the zero-padded range spectrum modulus) / os_range, then the
 * grid bin minimising sum_q (sensed_range(x) - r_hat_q)^2 (first minimum),
 * evaluated in fp64 exactly as the reference. frames complex64 [T][P][N];
 * rhat_d fp64 [T][P] (output, nullable); idx int64 [T]; res fp64 [T]. */
int gh_indirect_argmin_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                         const float* frames_d, int32_t n_trials, double* rhat_d,
                         int64_t* idx_d, double* res_d);
/* multilaterate_location alone, from caller range estimates rhat_d [T][P]. */
int gh_multilaterate_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                       const double* rhat_d, int32_t n_trials, int64_t* idx_d,
                       double* res_d);

/* ---- GHT1 hop-table container ------------------------------------------
 * save_hop_table / load_hop_table (src/interp.cpp:225-389, format
 * include/gridhop/interp.hpp:69-77): little-endian magic "GHT1", u32
 * version (1) / Q / bins / K / os / Ms, u64 scene hash, f64 worst residual,
 * then per bin per pair K u32 indices and K (re, im) f64 pairs. Errors are
 * GH_ERUNTIME with the reference's messages ("<path>: bad magic (not a GHT1
 * hop table)", "<path>: truncated ...", "<path>: stale hop table (scene or
 * grid mismatch)", ...). */
typedef struct gh_ght1_header {
  int32_t n_pairs;   /* Q: receivers of the reference, TX-RX pairs here */
  int32_t n_bins;
  int32_t k;         /* interpolation order 1..3 (polar tables store 3) */
  int32_t os_range;
  int32_t n_samples;
  uint64_t scene_hash;
  double max_residual;
} gh_ght1_header;

/* scene_hash (src/model.cpp:135-166): the reference's FNV-1a over the
 * receiver count, chirps, samples, f0, bandwidth, chirp duration, the TX
 * and every RX position (2-D, x then y). tx_xy[2], rx_xy[2 * n_rx]. */
uint64_t gh_scene_hash(int32_t n_rx, int32_t n_chirps, int32_t n_samples, double f0,
                       double bandwidth, double chirp_duration, const double* tx_xy,
                       const double* rx_xy);
/* Host arrays in the reference layout: idx u32 [bins][Q][K], coef f64
 * [bins][Q][K][2]. gh_ght1_read with idx = coef = NULL reads and validates
 * only the header; otherwise `capacity` (entries) must hold bins*Q*K. */
int gh_ght1_write(const char* path, const gh_ght1_header* hdr, const uint32_t* idx,
                  const double* coef);
int gh_ght1_read(const char* path, gh_ght1_header* hdr, uint32_t* idx, double* coef,
                 int64_t capacity);
/* Device tables: save downloads the operator; load validates the file
 * against the scene it is about to serve (hash, pairs, samples, os, bins:
 * "stale hop table") and uploads it. */
int gh_table_save(gh_table* t, const char* path, uint64_t scene_hash);
int gh_table_load(gh_ctx* ctx, const char* path, const gh_wave* wave, const gh_grid* grid,
                  uint64_t scene_hash, gh_table** out);

/* ---- stage kernels (device pointers) ---------------------------------- */
/* synthesize_frame + add_noise (src/synth.cpp:15-49) for trials
 * [trial0, trial0+T): frames complex64 [T][P][N]; truth fp64 [T][K][3]
 * (nullable). Same counter-based draws as the oracle. */
int gh_synth_d(gh_ctx* ctx, const gh_wave* wave, const gh_campaign* camp,
               uint64_t trial0, int32_t n_trials, int32_t wrap, float* frames_d,
               double* truth_d);
/* fast_time_spectra (src/hopping.cpp:121-129): zero-padded forward FFT,
 * complex64 [T][P][N] -> complex64 [T][P][M]. */
int gh_spectra_d(gh_ctx* ctx, const float* frames_d, int32_t n_trials,
                 int32_t n_pairs, int32_t n_samples, int32_t os_range,
                 float* spectra_d);
/* hop_decision_map (src/hopping.cpp:179-183), parity mode: complex64 frames
 * [T][P][N] -> fp32 maps [T][G]. */
int gh_hop_map_d(gh_ctx* ctx, gh_table* t, const float* frames_d,
                 int32_t n_trials, int32_t combine, float* map_d);
/* hop_estimate location stage (src/hopping.cpp:238-267) batched over
 * trials, FFT -> gather -> argmax fused: per-trial bin index (first strict
 * maximum, argmax_index src/direct.cpp:55-62) and its value. */
int gh_hop_argmax_d(gh_ctx* ctx, gh_table* t, const float* frames_d,
                    int32_t n_trials, int32_t combine, int64_t* idx_d,
                    float* val_d);
/* Same, from HOST complex128 frames [T][P][N] (the reference's FrameSet
 * element type) to HOST results; copies are inside the call. */
int gh_hop_estimate(gh_ctx* ctx, gh_table* t, const double* frames,
                    int32_t n_trials, int32_t combine, int64_t* idx,
                    double* val);
/* Multi-target form from HOST complex128 frames (BASELINE c3): the top-k
 * local maxima of gh_hop_topk_d, idx int64 [T][k] (-1 = none), val fp64
 * [T][k]; copies are inside the call, pipelined with the compute. */
int gh_hop_estimate_topk(gh_ctx* ctx, gh_table* t, const double* frames, int32_t n_trials,
                         int32_t combine, int32_t k, int64_t* idx, double* val);
/* Monte-Carlo campaign step (src/montecarlo.cpp:140-175, hop arm): synth
 * fused into the FFT, then gather + argmax; nothing but results touch HBM. */
int gh_campaign_hop_d(gh_ctx* ctx, gh_table* t, const gh_campaign* camp,
                      uint64_t trial0, int32_t n_trials, int32_t combine,
                      int64_t* idx_d, float* val_d);
/* Multi-target peak pick (BASELINE c3): per trial the k <= 8 best local
 * maxima of the hop map (a bin beats every smaller-index neighbour strictly
 * and every larger-index neighbour or ties; 8-neighbourhood in 2-D, 26 in
 * 3-D), ranked by (value desc, bin asc). idx_d int64 [T][k] (-1 = none),
 * val_d fp32 [T][k]. Campaign form synthesises the trials on the device. */
int gh_hop_topk_d(gh_ctx* ctx, gh_table* t, const float* frames_d, int32_t n_trials,
                  int32_t combine, int32_t k, int64_t* idx_d, float* val_d);
int gh_campaign_hop_topk_d(gh_ctx* ctx, gh_table* t, const gh_campaign* camp, uint64_t trial0,
                           int32_t n_trials, int32_t combine, int32_t k, int64_t* idx_d,
                           float* val_d);
/* The same peak pick on caller-provided maps fp32 [T][G] (e.g. direct maps). */
int gh_topk_local_max_d(gh_ctx* ctx, const gh_grid* grid, const float* map_d, int32_t n_trials,
                        int32_t k, int64_t* idx_d, float* val_d);
/* location_decision_map (src/direct.cpp:90-144) for T trials at once as the
 * complex contraction Z_p = Y_p (T x N) . A_p^H (N x G) on the tensor cores
 * (tcgen05, 3xTF32), |.|^2 summed over pairs in the epilogue. */
int gh_direct_map_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                    const float* frames_d, int32_t n_trials, int32_t combine,
                    float* map_d);
/* direct_estimate location stage (src/direct.cpp:230-239): per-trial argmax
 * fused into the contraction epilogue. */
int gh_direct_argmax_d(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid,
                       const float* frames_d, int32_t n_trials, int32_t combine,
                       int64_t* idx_d, float* val_d);

/* ---- host-buffer stage entry points ---------------------------------------
 * The reference signatures of the C++ wrappers (gridhop_b200.hpp) on HOST
 * complex128 arrays (the reference's CMat element type); the computation is
 * the device path of the _d forms (fp32 spectra and maps, fp64 table fits).
 *   gh_spectra          fast_time_spectra (hopping.hpp:14): [T][P][N] -> [T][P][M]
 *   gh_hop_map          hop_decision_map (hopping.hpp:22): -> map fp64 [T][G]
 *   gh_direct_map       location_decision_map (direct.hpp:19-23)
 *   gh_direct_estimate  direct_estimate location stage (direct.hpp:37-39)
 *   gh_synth            synthesize_frame + add_noise (synth.hpp:26-36) of the
 *                       campaign scene model; truth fp64 [T][K][3] (nullable)
 *   gh_add_noise        add_noise (synth.hpp:29-36): the per-(trial, pair)
 *                       substream draws, sigma = 10^(-snr/20); snr NaN: none
 *   gh_fit_atom         fit_atom (interp.hpp:41) of n ranges: idx [n][3],
 *                       coef complex128 [n][3], residual [n] (unused slots 0)
 *   gh_table_geometry   the table's n_samples, os_range and B / c           */
int gh_table_geometry(const gh_table* t, int32_t* n_samples, int32_t* os_range,
                      double* range_scale);
int gh_spectra(gh_ctx* ctx, const double* frames, int32_t n_trials, int32_t n_pairs,
               int32_t n_samples, int32_t os_range, double* spectra);
int gh_hop_map(gh_ctx* ctx, gh_table* t, const double* frames, int32_t n_trials, int32_t combine,
               double* map);
int gh_direct_map(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid, const double* frames,
                  int32_t n_trials, int32_t combine, double* map);
int gh_direct_estimate(gh_ctx* ctx, const gh_wave* wave, const gh_grid* grid, const double* frames,
                       int32_t n_trials, int32_t combine, int64_t* idx, double* val);
int gh_synth(gh_ctx* ctx, const gh_wave* wave, const gh_campaign* camp, uint64_t trial0,
             int32_t n_trials, int32_t wrap, double* frames, double* truth);
int gh_add_noise(gh_ctx* ctx, double* frames, int32_t n_trials, int32_t n_pairs, int32_t n_samples,
                 uint64_t seed, uint64_t trial0, double snr_db);
int gh_fit_atom(gh_ctx* ctx, int32_t n_samples, int32_t os_range, const double* r, int32_t n,
                int32_t scheme, uint32_t* idx, double* coef, double* residual);

/* ---- multi-GPU communicator ---------------------------------------------
 * One process per GPU. Rank 0 creates an id (ncclGetUniqueId), the caller
 * sends it to the other ranks (e.g. torch.distributed broadcast), and every
 * rank calls gh_comm_init with it (ncclCommInitRank) on its own context.
 * NCCL (libnccl.so.2) is loaded at run time: without it these calls fail
 * with GH_ERUNTIME and single-GPU campaigns still run (comm = NULL). */
typedef struct gh_comm gh_comm;
#define GH_COMM_ID_BYTES 128
int gh_comm_unique_id(uint8_t id[GH_COMM_ID_BYTES]);
int gh_comm_init(gh_ctx* ctx, const uint8_t id[GH_COMM_ID_BYTES], int32_t n_ranks, int32_t rank,
                 gh_comm** out);
int gh_comm_info(const gh_comm* comm, int32_t* n_ranks, int32_t* rank);
int gh_comm_destroy(gh_comm* comm);

/* ---- Monte-Carlo campaign driver ----------------------------------------
 * run_monte_carlo (src/montecarlo.cpp:99-179) on the device: for every
 * density (one hop table each, built on the device; LocationGrid::build's
 * axis count at spacing / density over the grid's extent, model.cpp:91-105),
 * every SNR and every algorithm, the campaign's n_trials trials — sharded
 * over the communicator's ranks in contiguous blocks, each trial keyed by
 * (seed, global trial) so estimates do not depend on the rank count — run
 * synthesis, the estimator and the statistics on the device. A trial's
 * estimates (topk per trial: argmax or the k best local maxima) are assigned
 * to its targets by the permutation of least total squared distance; the
 * cell counts hits per threshold (hit_ratio, montecarlo.cpp:181-190), the
 * squared-error sum (RMSE) and half-resolution hits. Cell vectors are summed
 * over ranks with one NCCL all-reduce. Optional CSVs follow write_trial_csv /
 * write_summary_csv (montecarlo.cpp:230-284; one trial row per target, v =
 * 0 as the campaign has no slow-time axis; written by rank 0).
 * Algorithm ids follow the reference's enum order (scenario.hpp:12). */
enum gh_algorithm { GH_ALGO_INDIRECT = 0, GH_ALGO_DIRECT = 1, GH_ALGO_HOP = 2 };
#define GH_MAX_THRESHOLDS 32
typedef struct {
  gh_wave wave;               /* waveform + TX-RX pairs                      */
  gh_grid grid;               /* location grid at density 1                  */
  gh_campaign scene;          /* truth / amplitude / SNR model               */
  int32_t scheme;             /* hop table interpolation scheme              */
  int32_t wrap;               /* 0: the reference's window checks           */
  int32_t combine;            /* GH_POWER / GH_MAGNITUDE                     */
  int32_t n_algorithms;
  const int32_t* algorithms;  /* gh_algorithm values, in record order        */
  int32_t n_snr;              /* 0: the scene's own SNR model, one cell      */
  const double* snr_db;       /* per-cell SNR (fixed mode); NaN = noiseless  */
  int32_t n_density;          /* 0: density 1                                */
  const double* density;
  int32_t n_thresholds;       /* 0: 0.2, 0.4 .. 3.0 m (scenario.cpp:177-179) */
  const double* thresholds_m;
  int64_t n_trials;           /* per cell, whole job                         */
  int32_t topk;               /* estimates per trial (<= 6 for statistics)   */
  int32_t batch;              /* trials per device batch, 0: automatic       */
  const char* trial_csv;      /* nullable                                    */
  const char* summary_csv;    /* nullable                                    */
  /* TableSource (montecarlo.hpp:43-45): when set, supplies the hop table of
   * each density (e.g. a GHT1 file through gh_table_load) instead of the
   * device build; the caller keeps ownership; *offline_ns is reported as the
   * cell's table acquisition time. */
  gh_table* (*table_source)(void* user, double density, const gh_grid* grid,
                            int64_t* offline_ns);
  void* table_source_user;
} gh_campaign_desc;
typedef struct {
  int32_t algorithm, density_idx, snr_idx, n_thresholds;
  double density, snr_db;     /* snr_db NaN: noiseless / per-pair model      */
  int64_t trials;             /* trials of the cell (all ranks)              */
  int64_t estimates;          /* scored (trial, target) pairs                */
  double thresholds_m[GH_MAX_THRESHOLDS];
  double hits[GH_MAX_THRESHOLDS];
  double hit_ratio[GH_MAX_THRESHOLDS];
  double hits_half_res;       /* within half a range resolution c / (4 B)    */
  double sq_err_sum, err_sum, rmse_m;
  double online_ms;           /* device time of the estimator, max over ranks */
  double offline_ms;          /* hop table build of the density (hop cells)  */
  double mean_online_ns;      /* online_ms per trial of the largest shard    */
} gh_cell_stats;
int gh_campaign_run(gh_ctx* ctx, gh_comm* comm, const gh_campaign_desc* desc, gh_cell_stats* out,
                    int32_t capacity, int32_t* n_cells);

#ifdef __cplusplus
}
#endif
#endif
