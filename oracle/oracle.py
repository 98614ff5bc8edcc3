"""ctypes front-end of the fp64 CPU oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs as the checker and the CPU
baseline. The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

_lib = None


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build() -> Path:
    src = HERE / "gridhop_oracle.cpp"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        from paper_2307_16550_b200.scene import CCampaign, CGrid, CWave  # plain ctypes structs
        L = C.CDLL(str(LIB))
        vp, i32, i64, u64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
        P = C.POINTER
        sig = {
            "or_last_error": (C.c_char_p, []),
            "or_splitmix64": (u64, [u64]),
            "or_substream": (u64, [u64, u64, u64]),
            "or_uniform": (f64, [u64, u64]),
            "or_sensed_range": (f64, [f64, vp, vp, vp, P(C.c_int)]),
            "or_grid_point": (None, [P(CGrid), i64, vp]),
            "or_scheme_order": (C.c_int, [C.c_int]),
            "or_fit_atom": (C.c_int, [C.c_int, C.c_int, f64, C.c_int, vp, vp, vp]),
            "or_build_table": (C.c_int, [P(CWave), P(CGrid), C.c_int, C.c_int, C.c_int, vp, vp, vp]),
            "or_scene_sample": (C.c_int, [P(CWave), P(CCampaign), u64, vp, vp, vp]),
            "or_synth": (C.c_int, [P(CWave), P(CCampaign), u64, i32, C.c_int, vp, vp]),
            "or_spectra": (C.c_int, [vp, i64, i32, i32, vp]),
            "or_hop_map": (C.c_int, [vp, i32, i32, i32, vp, vp, i64, i32, C.c_int, vp]),
            "or_direct_map": (C.c_int, [vp, i32, P(CWave), P(CGrid), C.c_int, C.c_int, vp]),
            "or_table_rows": (C.c_int, [P(CWave), P(CGrid), C.c_int, vp, i64, C.c_int, vp, vp]),
            "or_hop_map_onfly": (C.c_int, [vp, i32, P(CWave), P(CGrid), C.c_int, C.c_int, C.c_int,
                                           vp]),
            "or_argmax": (i64, [vp, i64]),
            "or_topk_local_max": (C.c_int, [vp, P(CGrid), i32, vp, vp]),
            "or_range_peaks": (C.c_int, [vp, i64, i32, i32, vp]),
            "or_hop_map_mc": (C.c_int, [vp, i32, i32, i32, i32, vp, vp, i64, i32, vp]),
            "or_hop_velocity": (C.c_int, [vp, i32, i32, P(CWave), P(CGrid), f64, f64, i32, i32,
                                          vp, vp, vp]),
            "or_direct_velocity": (C.c_int, [vp, i32, i32, P(CWave), P(CGrid), f64, f64, i32,
                                             vp, vp, vp]),
            "or_multilaterate": (C.c_int, [P(CWave), P(CGrid), vp, i32, C.c_int, vp, vp]),
            "or_campaign_hop": (C.c_int, [P(CWave), P(CGrid), P(CCampaign), vp, vp, i32, C.c_int,
                                          C.c_int, u64, i32, C.c_int, vp, vp]),
            "or_campaign_hop_topk": (C.c_int, [P(CWave), P(CGrid), P(CCampaign), vp, vp, i32,
                                               C.c_int, C.c_int, u64, i32, i32, C.c_int, vp, vp]),
            "or_trial_stats": (C.c_int, [P(CGrid), vp, i32, vp, i32, i32, vp, i32, f64, f64, vp,
                                         vp]),
            "or_campaign_direct": (C.c_int, [P(CWave), P(CGrid), P(CCampaign), C.c_int, C.c_int,
                                             u64, i32, C.c_int, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int) -> None:
    if st != 0:
        raise OracleError(st, lib().or_last_error().decode())


def nthreads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def fit_atom(n_samples: int, os_: int, r: float, scheme: int):
    idx = np.zeros(3, dtype=np.uint32)
    coef = np.zeros(6, dtype=np.float64)
    res = C.c_double()
    _check(lib().or_fit_atom(n_samples, os_, r, scheme, idx.ctypes.data, coef.ctypes.data,
                             C.byref(res)))
    k = {1: 1, 2: 2, 3: 3, 4: 3}[scheme]
    return idx[:k].copy(), coef.view(np.complex128)[:k].copy(), res.value


def sensed_range(scale: float, tx, rx, x) -> float:
    tx, rx, x = (np.ascontiguousarray(v, dtype=np.float64) for v in (tx, rx, x))
    st = C.c_int()
    r = lib().or_sensed_range(scale, tx.ctypes.data, rx.ctypes.data, x.ctypes.data, C.byref(st))
    _check(st.value)
    return r


def build_table(scene, scheme: int | None = None, wrap: bool | None = None, threads: int | None = None):
    scheme = scene.scheme if scheme is None else scheme
    k = {1: 1, 2: 2, 3: 3, 4: 3}[scheme]
    n = scene.n_bins * scene.n_pairs * k
    idx = np.zeros(n, dtype=np.uint32)
    coef = np.zeros(2 * n, dtype=np.float64)
    mr = C.c_double()
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().or_build_table(C.byref(w), C.byref(g), scheme,
                                int(scene.wrap if wrap is None else wrap),
                                threads or nthreads(), idx.ctypes.data, coef.ctypes.data, C.byref(mr)))
    shape = (scene.n_bins, scene.n_pairs, k)
    return idx.reshape(shape), coef.view(np.complex128).reshape(shape), mr.value


def scene_sample(scene, trial: int, snr_db=None):
    K, P = scene.n_targets, scene.n_pairs
    tg = np.zeros((K, 3)); al = np.zeros(2 * K * P); sg = np.zeros(P)
    w, c = scene.c_wave(), scene.c_campaign(snr_db)
    _check(lib().or_scene_sample(C.byref(w), C.byref(c), trial, tg.ctypes.data, al.ctypes.data,
                                 sg.ctypes.data))
    return tg, al.view(np.complex128).reshape(K, P), sg


def synth(scene, trial0: int, n_trials: int, snr_db=None, wrap: bool | None = None):
    """complex128 frames [T, P, N] and truth [T, K, 3]."""
    fr = np.zeros(n_trials * scene.n_pairs * scene.n_samples * 2)
    tr = np.zeros((n_trials, scene.n_targets, 3))
    w, c = scene.c_wave(), scene.c_campaign(snr_db)
    _check(lib().or_synth(C.byref(w), C.byref(c), trial0, n_trials,
                          int(scene.wrap if wrap is None else wrap), fr.ctypes.data, tr.ctypes.data))
    return fr.view(np.complex128).reshape(n_trials, scene.n_pairs, scene.n_samples), tr


def spectra(frames: np.ndarray, m: int) -> np.ndarray:
    frames = np.ascontiguousarray(frames, dtype=np.complex128)
    n = frames.shape[-1]
    rows = int(np.prod(frames.shape[:-1]))
    out = np.zeros(rows * m, dtype=np.complex128)
    _check(lib().or_spectra(frames.ctypes.data, rows, n, m, out.ctypes.data))
    return out.reshape(*frames.shape[:-1], m)


def hop_map(spec: np.ndarray, idx: np.ndarray, coef: np.ndarray, magnitude: bool = False):
    spec = np.ascontiguousarray(spec, dtype=np.complex128)
    T, P, M = spec.shape
    G, P2, K = idx.shape
    assert P2 == P
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    coef = np.ascontiguousarray(coef, dtype=np.complex128)
    out = np.zeros((T, G))
    _check(lib().or_hop_map(spec.ctypes.data, T, P, M, idx.ctypes.data, coef.ctypes.data, G, K,
                            int(magnitude), out.ctypes.data))
    return out


def hop_map_mc(spec: np.ndarray, idx: np.ndarray, coef: np.ndarray):
    """scan_planes over Mc chirps (power): spec complex [T, P, Mc, M]."""
    spec = np.ascontiguousarray(spec, dtype=np.complex128)
    T, P, Mc, M = spec.shape
    G, P2, K = idx.shape
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    coef = np.ascontiguousarray(coef, dtype=np.complex128)
    out = np.zeros((T, G))
    _check(lib().or_hop_map_mc(spec.ctypes.data, T, P, Mc, M, idx.ctypes.data, coef.ctypes.data, G, K,
                               out.ctypes.data))
    return out


def velocity(scene, frames: np.ndarray, loc: np.ndarray, doppler_scale: float, spacing: float,
             half: int, os_doppler: int = 1, method: str = "hop"):
    """hop_velocity / direct_velocity at the located bins: frames complex
    [T, P, Mc, N] -> (velocity-grid index [T], value [T])."""
    frames = np.ascontiguousarray(frames, dtype=np.complex128)
    T, P, Mc, N = frames.shape
    loc = np.ascontiguousarray(loc, dtype=np.int64)
    vidx = np.zeros(T, dtype=np.int64)
    vval = np.zeros(T)
    w, g = scene.c_wave(), scene.c_grid()
    if method == "hop":
        _check(lib().or_hop_velocity(frames.ctypes.data, T, Mc, C.byref(w), C.byref(g), doppler_scale,
                                     spacing, half, os_doppler, loc.ctypes.data, vidx.ctypes.data,
                                     vval.ctypes.data))
    else:
        _check(lib().or_direct_velocity(frames.ctypes.data, T, Mc, C.byref(w), C.byref(g),
                                        doppler_scale, spacing, half, loc.ctypes.data,
                                        vidx.ctypes.data, vval.ctypes.data))
    return vidx, vval


def table_rows(scene, bins: np.ndarray, scheme: int | None = None, threads: int | None = None):
    """or_table_rows: the mapping operator's rows for a subset of bins."""
    bins = np.ascontiguousarray(bins, dtype=np.int64)
    K = lib().or_scheme_order(scene.scheme if scheme is None else scheme)
    idx = np.zeros((bins.size, scene.n_pairs, K), dtype=np.uint32)
    coef = np.zeros((bins.size, scene.n_pairs, K), dtype=np.complex128)
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().or_table_rows(C.byref(w), C.byref(g), scene.scheme if scheme is None else scheme,
                               bins.ctypes.data, bins.size, threads or nthreads(), idx.ctypes.data,
                               coef.ctypes.data))
    return idx, coef


def hop_map_onfly(scene, spec: np.ndarray, magnitude: bool = False, threads: int | None = None):
    """or_hop_map_onfly: the hop map without a stored table (grids too large
    to tabulate on the host): complex spectra [T, P, M] -> [T, G]."""
    spec = np.ascontiguousarray(spec, dtype=np.complex128)
    T = spec.shape[0]
    out = np.zeros((T, scene.n_bins))
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().or_hop_map_onfly(spec.ctypes.data, T, C.byref(w), C.byref(g), scene.scheme,
                                  int(magnitude), threads or nthreads(), out.ctypes.data))
    return out


def direct_map(scene, frames: np.ndarray, magnitude: bool = False, threads: int | None = None):
    frames = np.ascontiguousarray(frames, dtype=np.complex128)
    T = frames.shape[0]
    out = np.zeros((T, scene.n_bins))
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().or_direct_map(frames.ctypes.data, T, C.byref(w), C.byref(g), int(magnitude),
                               threads or nthreads(), out.ctypes.data))
    return out


def argmax(v: np.ndarray) -> int:
    v = np.ascontiguousarray(v, dtype=np.float64)
    r = lib().or_argmax(v.ctypes.data, v.size)
    if r < 0:
        raise OracleError(1, lib().or_last_error().decode())
    return int(r)


def range_peaks(spec: np.ndarray, os_range: int) -> np.ndarray:
    """r_hat per row of complex spectra [..., M]: range_doppler_map +
    RangeDopplerMap::peak at Mc = 1 (src/indirect.cpp:10-56)."""
    spec = np.ascontiguousarray(spec, dtype=np.complex128)
    rows = int(np.prod(spec.shape[:-1]))
    out = np.zeros(rows)
    _check(lib().or_range_peaks(spec.ctypes.data, rows, spec.shape[-1], os_range, out.ctypes.data))
    return out.reshape(spec.shape[:-1])


def multilaterate(scene, rhat: np.ndarray, threads: int | None = None):
    """multilaterate_location (src/indirect.cpp:58-83): (idx [T], residual [T])."""
    rhat = np.ascontiguousarray(rhat, dtype=np.float64)
    T = rhat.shape[0]
    idx = np.zeros(T, dtype=np.int64)
    res = np.zeros(T)
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().or_multilaterate(C.byref(w), C.byref(g), rhat.ctypes.data, T, threads or nthreads(),
                                  idx.ctypes.data, res.ctypes.data))
    return idx, res


def topk_local_max(scene, m: np.ndarray, k: int):
    m = np.ascontiguousarray(m, dtype=np.float64)
    idx = np.zeros(k, dtype=np.int64); val = np.zeros(k)
    g = scene.c_grid()
    _check(lib().or_topk_local_max(m.ctypes.data, C.byref(g), k, idx.ctypes.data, val.ctypes.data))
    return idx, val


def campaign_hop(scene, idx, coef, trial0: int, n_trials: int, snr_db=None, magnitude=False,
                 wrap=None, threads: int | None = None):
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    coef = np.ascontiguousarray(coef, dtype=np.complex128)
    K = idx.shape[-1]
    ei = np.zeros(n_trials, dtype=np.int64); ev = np.zeros(n_trials)
    w, g, c = scene.c_wave(), scene.c_grid(), scene.c_campaign(snr_db)
    _check(lib().or_campaign_hop(C.byref(w), C.byref(g), C.byref(c), idx.ctypes.data,
                                 coef.ctypes.data, K, int(magnitude),
                                 int(scene.wrap if wrap is None else wrap), trial0, n_trials,
                                 threads or nthreads(), ei.ctypes.data, ev.ctypes.data))
    return ei, ev


def campaign_direct(scene, trial0: int, n_trials: int, snr_db=None, magnitude=False, wrap=None,
                    threads: int | None = None):
    ei = np.zeros(n_trials, dtype=np.int64); ev = np.zeros(n_trials)
    w, g, c = scene.c_wave(), scene.c_grid(), scene.c_campaign(snr_db)
    _check(lib().or_campaign_direct(C.byref(w), C.byref(g), C.byref(c), int(magnitude),
                                    int(scene.wrap if wrap is None else wrap), trial0, n_trials,
                                    threads or nthreads(), ei.ctypes.data, ev.ctypes.data))
    return ei, ev


def campaign_hop_topk(scene, idx, coef, trial0: int, n_trials: int, topk: int, snr_db=None,
                      magnitude=False, wrap=None, threads: int | None = None):
    """Top-k local maxima per trial of the hop map (BASELINE c3/c5): (idx [T, k], val [T, k])."""
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    coef = np.ascontiguousarray(coef, dtype=np.complex128)
    K = idx.shape[-1]
    ei = np.zeros((n_trials, topk), dtype=np.int64)
    ev = np.zeros((n_trials, topk))
    w, g, c = scene.c_wave(), scene.c_grid(), scene.c_campaign(snr_db)
    _check(lib().or_campaign_hop_topk(C.byref(w), C.byref(g), C.byref(c), idx.ctypes.data,
                                      coef.ctypes.data, K, int(magnitude),
                                      int(scene.wrap if wrap is None else wrap), trial0, n_trials,
                                      topk, threads or nthreads(), ei.ctypes.data, ev.ctypes.data))
    return ei, ev


DEFAULT_THRESHOLDS = tuple(0.2 * i for i in range(1, 16))  # scenario.cpp:177-179


def half_resolution(scene) -> float:
    """Half the range resolution c / (2 B) (model.hpp range_resolution)."""
    return 0.5 * scene.c / (2.0 * scene.bandwidth)


def miss_distance(scene) -> float:
    """Distance charged to an unmatched target: the grid box diagonal."""
    sp = np.asarray(scene.grid_spacing, dtype=np.float64)
    n = np.asarray(scene.grid_n, dtype=np.float64)
    return float(np.sqrt(np.sum((sp * n) ** 2)))


def trial_stats(scene, est: np.ndarray, truth: np.ndarray, thresholds=DEFAULT_THRESHOLDS):
    """or_trial_stats: (stats vector [4 + nth], assignment [T, kt]). est [T]
    or [T, ke] grid bins (-1 = none); truth [T, kt, 3]."""
    est = np.ascontiguousarray(est, dtype=np.int64)
    if est.ndim == 1:
        est = est[:, None]
    truth = np.ascontiguousarray(truth, dtype=np.float64)
    T, ke = est.shape
    kt = truth.shape[1]
    th = np.ascontiguousarray(thresholds, dtype=np.float64)
    out = np.zeros(4 + th.size)
    assign = np.zeros((T, kt), dtype=np.int32)
    g = scene.c_grid()
    _check(lib().or_trial_stats(C.byref(g), est.ctypes.data, ke, truth.ctypes.data, kt, T,
                                th.ctypes.data, th.size, half_resolution(scene),
                                miss_distance(scene), out.ctypes.data, assign.ctypes.data))
    return out, assign
