/*
 * gridhop_oracle.h — CPU fp64 restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker for the
 * B200 path and the CPU baseline timed by bench.py's `cpu_baseline` leg and
 * `--impl reference` arm. Only tests/, __graft_entry__.smoke() and bench.py
 * may load it; the product library (paper_2307_16550_b200) never links or
 * calls it.
 *
 * Every function restates a reference function (file:line under
 * /root/reference/proj/core); the reference itself cannot be built here
 * (Eigen3 + FFTW3 absent), so this restatement is
 * pinned against the reference's own known-answer tests (tests/golden/,
 * tests/test_oracle_golden.py) and cross-checked by an independent numpy
 * restatement (oracle/oracle_np.py).
 *
 * Plain C ABI (extern "C"), caller-owned buffers, int status:
 *   0 ok, 1 invalid_argument, 2 runtime_error, 3 domain_error
 * with the message from or_last_error() — the same convention as the
 * product's gh_* ABI, mirroring the reference's exception types.
 */
#ifndef GRIDHOP_ORACLE_H
#define GRIDHOP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Waveform + TX/RX pair geometry. The reference has one TX and Q RX
 * (model.hpp:44-50); a pair list generalises it (BASELINE c3-c5 use several
 * TX). Positions are 3-D; 2-D scenes set z = 0 (sqrt(dx²+dy²+0) rounds
 * exactly like the reference's 2-D norm). */
typedef struct {
  int32_t n_samples;   /* N, fast-time samples per pair (model.hpp:26)     */
  int32_t os_range;    /* M / N, zero-padding factor (interp.hpp:47)       */
  double range_scale;  /* B / c, fast-time bins per metre (model.hpp:36)   */
  int32_t n_pairs;     /* P                                                */
  const double* tx;    /* [P][3]                                           */
  const double* rx;    /* [P][3]                                           */
} or_wave;

/* Lattice, x fastest then y then z (model.hpp:77-92, model.cpp:108-111). */
typedef struct {
  double origin[3];
  double spacing[3];
  int32_t n[3];
} or_grid;

/* Monte-Carlo trial scene model (montecarlo.cpp:48-66 + BASELINE
 * extensions: K targets, per-pair amplitudes and SNR). */
typedef struct {
  uint64_t seed;
  int32_t n_targets;
  int32_t dims;          /* 2 or 3 position draws per target              */
  double area_lo[3];
  double area_hi[3];
  int32_t amp_mode;      /* 0 unit-phase shared (reference), 1 unit-phase
                            per pair, 2 CN(0,1) shared, 3 CN(0,1) per pair */
  int32_t snr_mode;      /* 0 fixed snr_db, 1 U[snr_lo, snr_hi] per pair,
                            2 noiseless                                   */
  double snr_db;
  double snr_lo;
  double snr_hi;
} or_campaign;

enum { OR_NEAREST = 1, OR_LINEAR = 2, OR_POLY3 = 3, OR_POLAR = 4 };

const char* or_last_error(void);

/* rng.hpp:11-52 restated with a counter-addressable SplitMix64 stream. */
uint64_t or_splitmix64(uint64_t x);
uint64_t or_substream(uint64_t seed, uint64_t a, uint64_t b);
double or_uniform(uint64_t key, uint64_t counter);

double or_sensed_range(double range_scale, const double* tx, const double* rx,
                       const double* x, int* status);
void or_grid_point(const or_grid* g, int64_t k, double* out3);

int or_scheme_order(int scheme);
int or_fit_atom(int n_samples, int os, double r, int scheme, uint32_t* idx3,
                double* coef6, double* residual);
int or_build_table(const or_wave* w, const or_grid* g, int scheme, int wrap,
                   int n_threads, uint32_t* idx, double* coef,
                   double* max_residual);

/* Rows of the mapping operator for a subset of bins (or_build_table's
 * per-entry fit, interp.cpp:156-223), wrap mode: idx [n][P][K], coef
 * [n][P][K][2]. For grids too large to tabulate on the host (c5). */
int or_table_rows(const or_wave* w, const or_grid* g, int scheme, const int64_t* bins,
                  int64_t n, int n_threads, uint32_t* idx, double* coef);
/* The hop map (hop_map_trial's arithmetic, hopping.cpp:59-102) with every
 * (bin, pair) fitted on the fly instead of read from a stored table, bins
 * parallel over threads: spectra [T][P][M][2] -> map [T][G]. */
int or_hop_map_onfly(const double* spectra, int32_t n_trials, const or_wave* w,
                     const or_grid* g, int scheme, int magnitude, int n_threads, double* map);

int or_scene_sample(const or_wave* w, const or_campaign* c, uint64_t trial,
                    double* targets /*[K][3]*/, double* alpha /*[K][P][2]*/,
                    double* sigma /*[P]*/);
int or_synth(const or_wave* w, const or_campaign* c, uint64_t trial0,
             int32_t n_trials, int wrap, double* frames /*[T][P][N][2]*/,
             double* truth /*[T][K][3] or NULL*/);

int or_spectra(const double* frames, int64_t rows, int32_t n, int32_t m,
               double* out /*[rows][m][2]*/);
int or_hop_map(const double* spectra, int32_t n_trials, int32_t n_pairs,
               int32_t m, const uint32_t* idx, const double* coef,
               int64_t n_bins, int32_t k, int magnitude, double* map);
int or_hop_map_mc(const double* spectra, int32_t n_trials, int32_t n_pairs, int32_t n_chirps,
                  int32_t m, const uint32_t* idx, const double* coef, int64_t n_bins, int32_t k,
                  double* map);
int or_direct_map(const double* frames, int32_t n_trials, const or_wave* w,
                  const or_grid* g, int magnitude, int n_threads, double* map);
int64_t or_argmax(const double* v, int64_t n);
/* Velocity stage at located bins (hopping.cpp:185-236, direct.cpp:145-228):
 * frames [T][P][Mc][N][2]; VelocityGrid (spacing, half); os_d >= 1. */
int or_hop_velocity(const double* frames, int32_t n_trials, int32_t n_chirps, const or_wave* w,
                    const or_grid* g, double doppler_scale, double spacing, int32_t half,
                    int32_t os_d, const int64_t* loc, int64_t* vidx, double* vval);
int or_direct_velocity(const double* frames, int32_t n_trials, int32_t n_chirps, const or_wave* w,
                       const or_grid* g, double doppler_scale, double spacing, int32_t half,
                       const int64_t* loc, int64_t* vidx, double* vval);
/* Indirect pipeline, location stage (src/indirect.cpp:10-83, Mc = 1). */
int or_range_peaks(const double* spectra, int64_t rows, int32_t m, int32_t os_range,
                   double* rhat);
int or_multilaterate(const or_wave* w, const or_grid* g, const double* rhat, int32_t n_trials,
                     int n_threads, int64_t* idx, double* residual);
int or_topk_local_max(const double* map, const or_grid* g, int32_t k,
                      int64_t* idx_out, double* val_out);

/* Whole-trial CPU pipelines (the CPU baseline): synth -> spectra -> hop map
 * -> argmax per trial, parallel_for over trials (montecarlo.cpp:140). */
int or_campaign_hop(const or_wave* w, const or_grid* g, const or_campaign* c,
                    const uint32_t* idx, const double* coef, int32_t k,
                    int magnitude, int wrap, uint64_t trial0, int32_t n_trials,
                    int n_threads, int64_t* est_idx, double* est_val);
int or_campaign_hop_topk(const or_wave* w, const or_grid* g, const or_campaign* c,
                         const uint32_t* idx, const double* coef, int32_t k, int magnitude,
                         int wrap, uint64_t trial0, int32_t n_trials, int32_t topk,
                         int n_threads, int64_t* est_idx, double* est_val);
/* Campaign statistics of a batch (hit_ratio, montecarlo.cpp:181-190, + RMSE
 * and K-target assignment); see the definition for the layout of out. */
int or_trial_stats(const or_grid* g, const int64_t* est, int32_t ke, const double* truth,
                   int32_t kt, int32_t n_trials, const double* thresholds, int32_t nth,
                   double half_res, double miss_m, double* out, int32_t* assign);
int or_campaign_direct(const or_wave* w, const or_grid* g, const or_campaign* c,
                       int magnitude, int wrap, uint64_t trial0,
                       int32_t n_trials, int n_threads, int64_t* est_idx,
                       double* est_val);

#ifdef __cplusplus
}
#endif
#endif
