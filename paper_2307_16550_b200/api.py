"""Python host mirror of the reference estimator interfaces over the C ABI.

Names follow the reference library (include/gridhop/{hopping,direct,interp,
synth,montecarlo}.hpp); arrays on the device are torch tensors (torch is
only the device-memory / stream plumbing), host arrays are numpy. Every call
goes through libgridhop_b200.so; there is no CPU fallback — a missing or
unloadable library raises at import time.

Error behaviour mirrors the reference's exception types:
  GH_EINVAL   -> InvalidArgument (ValueError)      std::invalid_argument
  GH_ERUNTIME -> GridhopRuntimeError (RuntimeError) std::runtime_error
  GH_EDOMAIN  -> DomainError (ArithmeticError)      std::domain_error
  GH_ECUDA    -> CudaError (RuntimeError)
"""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

import numpy as np

from .scene import CCampaign, CGrid, CWave, Scene, POWER

LIB_PATH = Path(__file__).resolve().parent / "libgridhop_b200.so"
HEADER = Path(__file__).resolve().parent.parent / "include" / "gridhop_b200.h"


class InvalidArgument(ValueError):
    pass


class GridhopRuntimeError(RuntimeError):
    pass


class DomainError(ArithmeticError):
    pass


class CudaError(RuntimeError):
    pass


_EXC = {1: InvalidArgument, 2: GridhopRuntimeError, 3: DomainError, 4: CudaError}


class VelocityGridC(C.Structure):
    """gh_velocity_grid: VelocityGrid (model.hpp:93-107) + doppler_scale."""
    _fields_ = [("doppler_scale", C.c_double), ("spacing", C.c_double), ("half", C.c_int32),
                ("os_doppler", C.c_int32)]


def velocity_grid(f0: float, chirp_duration: float, n_chirps: int, speed_bound: float,
                  density: float, os_doppler: int = 1, c: float = 299792458.0) -> VelocityGridC:
    """VelocityGrid::build (model.cpp:116-125) and doppler_scale (model.hpp:38-40)."""
    if not (density > 0):
        raise InvalidArgument("velocity grid: density must be positive")
    if not (speed_bound > 0):
        raise InvalidArgument("velocity grid: speed bound must be positive")
    speed_res = c / (2.0 * f0 * chirp_duration * n_chirps)
    spacing = speed_res / density
    half = int(np.floor(speed_bound / spacing + 1e-9))
    return VelocityGridC(f0 * chirp_duration * n_chirps / c, spacing, half, os_doppler)


class Mrf1Header(C.Structure):
    """gh_mrf1_header: the MRF1 capture header (frame_io.hpp:10-16)."""
    _fields_ = [("n_rx", C.c_int32), ("n_chirps", C.c_int32), ("n_samples", C.c_int32),
                ("n_frames", C.c_int32), ("f0", C.c_double), ("bandwidth", C.c_double),
                ("chirp_duration", C.c_double), ("tx", C.c_double * 2)]


class Ght1Header(C.Structure):
    """gh_ght1_header: the GHT1 container header (interp.hpp:69-71)."""
    _fields_ = [("n_pairs", C.c_int32), ("n_bins", C.c_int32), ("k", C.c_int32),
                ("os_range", C.c_int32), ("n_samples", C.c_int32), ("scene_hash", C.c_uint64),
                ("max_residual", C.c_double)]

MAX_THRESHOLDS = 32
ALGO_INDIRECT, ALGO_DIRECT, ALGO_HOP = 0, 1, 2  # Algorithm (scenario.hpp:12)
ALGO_IDS = {"indirect": ALGO_INDIRECT, "direct": ALGO_DIRECT, "hop": ALGO_HOP}


class CampaignDesc(C.Structure):
    """gh_campaign_desc: a Scenario (scenario.hpp:22-52) for the device driver."""
    _fields_ = [("wave", CWave), ("grid", CGrid), ("scene", CCampaign), ("scheme", C.c_int32),
                ("wrap", C.c_int32), ("combine", C.c_int32), ("n_algorithms", C.c_int32),
                ("algorithms", C.POINTER(C.c_int32)), ("n_snr", C.c_int32),
                ("snr_db", C.POINTER(C.c_double)), ("n_density", C.c_int32),
                ("density", C.POINTER(C.c_double)), ("n_thresholds", C.c_int32),
                ("thresholds_m", C.POINTER(C.c_double)), ("n_trials", C.c_int64),
                ("topk", C.c_int32), ("batch", C.c_int32), ("trial_csv", C.c_char_p),
                ("summary_csv", C.c_char_p), ("table_source", C.c_void_p),
                ("table_source_user", C.c_void_p)]


class CellStats(C.Structure):
    """gh_cell_stats: one (density, SNR, algorithm) cell of a campaign."""
    _fields_ = [("algorithm", C.c_int32), ("density_idx", C.c_int32), ("snr_idx", C.c_int32),
                ("n_thresholds", C.c_int32), ("density", C.c_double), ("snr_db", C.c_double),
                ("trials", C.c_int64), ("estimates", C.c_int64),
                ("thresholds_m", C.c_double * MAX_THRESHOLDS),
                ("hits", C.c_double * MAX_THRESHOLDS), ("hit_ratio", C.c_double * MAX_THRESHOLDS),
                ("hits_half_res", C.c_double), ("sq_err_sum", C.c_double), ("err_sum", C.c_double),
                ("rmse_m", C.c_double), ("online_ms", C.c_double), ("offline_ms", C.c_double),
                ("mean_online_ns", C.c_double)]


_lib = None


def exported_symbols() -> list[str]:
    """Function names declared in include/gridhop_b200.h."""
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"\b(gh_[a-z0-9_]+)\s*\(", txt)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        path = Path(os.environ.get("GH_LIB_PATH", LIB_PATH))  # diagnostic builds (tools/)
        if not path.exists():
            raise ImportError(f"{path} is missing: run __graft_entry__.build()")
        L = C.CDLL(str(path))
        vp, i32, i64, u64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
        P = C.POINTER
        sig = {
            "gh_last_error": (C.c_char_p, []),
            "gh_abi_version": (C.c_int, []),
            "gh_ctx_create": (C.c_int, [i32, P(vp)]),
            "gh_ctx_destroy": (C.c_int, [vp]),
            "gh_ctx_get_stream": (C.c_int, [vp, P(vp)]),
            "gh_ctx_set_stream": (C.c_int, [vp, vp]),
            "gh_ctx_synchronize": (C.c_int, [vp]),
            "gh_ctx_launch_count": (C.c_int, [vp, P(i64)]),
            "gh_ctx_set_timing": (C.c_int, [vp, i32]),
            "gh_ctx_kernel_time": (C.c_int, [vp, C.c_char_p, P(f64), P(i64)]),
            "gh_ctx_reset_timing": (C.c_int, [vp]),
            "gh_measure_smem_peak": (C.c_int, [vp, P(f64)]),
            "gh_ctx_set_direct_impl": (C.c_int, [vp, i32]),
            "gh_ctx_set_topk_impl": (C.c_int, [vp, i32]),
            "gh_ctx_set_debug_checks": (C.c_int, [vp, i32]),
            "gh_table_build": (C.c_int, [vp, P(CWave), P(CGrid), i32, i32, P(vp)]),
            "gh_table_upload": (C.c_int, [vp, P(CWave), P(CGrid), i32, vp, vp, P(vp)]),
            "gh_table_build_shard": (C.c_int, [vp, P(CWave), P(CGrid), i32, i32, i32, i32, P(vp)]),
            "gh_table_info": (C.c_int, [vp, P(i64), P(i32), P(i32), P(i32), P(f64)]),
            "gh_table_download": (C.c_int, [vp, vp, vp]),
            "gh_table_rows": (C.c_int, [vp, vp, i64, vp, vp]),
            "gh_table_set_core": (C.c_int, [vp, i32, i32]),
            "gh_table_destroy": (C.c_int, [vp]),
            "gh_synth_d": (C.c_int, [vp, P(CWave), P(CCampaign), u64, i32, i32, vp, vp]),
            "gh_spectra_d": (C.c_int, [vp, vp, i32, i32, i32, i32, vp]),
            "gh_hop_map_d": (C.c_int, [vp, vp, vp, i32, i32, vp]),
            "gh_hop_argmax_d": (C.c_int, [vp, vp, vp, i32, i32, vp, vp]),
            "gh_hop_estimate": (C.c_int, [vp, vp, vp, i32, i32, vp, vp]),
            "gh_hop_estimate_topk": (C.c_int, [vp, vp, vp, i32, i32, i32, vp, vp]),
            "gh_campaign_hop_d": (C.c_int, [vp, vp, P(CCampaign), u64, i32, i32, vp, vp]),
            "gh_hop_topk_d": (C.c_int, [vp, vp, vp, i32, i32, i32, vp, vp]),
            "gh_campaign_hop_topk_d": (C.c_int, [vp, vp, P(CCampaign), u64, i32, i32, i32, vp, vp]),
            "gh_topk_local_max_d": (C.c_int, [vp, P(CGrid), vp, i32, i32, vp, vp]),
            "gh_direct_map_d": (C.c_int, [vp, P(CWave), P(CGrid), vp, i32, i32, vp]),
            "gh_direct_argmax_d": (C.c_int, [vp, P(CWave), P(CGrid), vp, i32, i32, vp, vp]),
            "gh_scene_hash": (u64, [i32, i32, i32, f64, f64, f64, vp, vp]),
            "gh_indirect_argmin_d": (C.c_int, [vp, P(CWave), P(CGrid), vp, i32, vp, vp, vp]),
            "gh_hop_map_mc_d": (C.c_int, [vp, vp, vp, i32, i32, vp]),
            "gh_hop_velocity_d": (C.c_int, [vp, P(CWave), P(CGrid), P(VelocityGridC), vp, i32, i32,
                                            vp, vp, vp]),
            "gh_direct_velocity_d": (C.c_int, [vp, P(CWave), P(CGrid), P(VelocityGridC), vp, i32,
                                               i32, vp, vp, vp]),
            "gh_hop_argmax_mc_d": (C.c_int, [vp, vp, vp, i32, i32, vp, vp]),
            "gh_mrf1_write": (C.c_int, [C.c_char_p, P(Mrf1Header), vp, vp]),
            "gh_mrf1_read": (C.c_int, [C.c_char_p, P(Mrf1Header), vp, i32, vp, i64]),
            "gh_multilaterate_d": (C.c_int, [vp, P(CWave), P(CGrid), vp, i32, vp, vp]),
            "gh_ght1_write": (C.c_int, [C.c_char_p, P(Ght1Header), vp, vp]),
            "gh_ght1_read": (C.c_int, [C.c_char_p, P(Ght1Header), vp, vp, i64]),
            "gh_table_save": (C.c_int, [vp, C.c_char_p, u64]),
            "gh_comm_unique_id": (C.c_int, [vp]),
            "gh_comm_init": (C.c_int, [vp, vp, i32, i32, P(vp)]),
            "gh_comm_info": (C.c_int, [vp, P(i32), P(i32)]),
            "gh_comm_destroy": (C.c_int, [vp]),
            "gh_campaign_run": (C.c_int, [vp, vp, P(CampaignDesc), P(CellStats), i32, P(i32)]),
            "gh_table_load": (C.c_int, [vp, C.c_char_p, P(CWave), P(CGrid), u64, P(vp)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        msg = lib().gh_last_error().decode()
        raise _EXC.get(status, RuntimeError)(msg)


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _torch():
    import torch
    return torch


class Context:
    """gh_ctx: one device, one stream, scratch buffers."""

    def __init__(self, device: int = 0, torch_stream: bool = True):
        h = C.c_void_p()
        _check(lib().gh_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        if torch_stream:
            # enqueue on torch's current stream so kernels are ordered with the
            # torch ops that produce inputs / consume outputs
            torch = _torch()
            s = torch.cuda.current_stream(device)
            _check(lib().gh_ctx_set_stream(h, C.c_void_p(s.cuda_stream)))
            self._torch_stream = s
        else:
            self._torch_stream = None

    def close(self) -> None:
        if self.h:
            _check(lib().gh_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream_ptr(self) -> int:
        s = C.c_void_p()
        _check(lib().gh_ctx_get_stream(self.h, C.byref(s)))
        return int(s.value or 0)

    def torch_stream(self):
        if self._torch_stream is not None:
            return self._torch_stream
        torch = _torch()
        return torch.cuda.ExternalStream(self.stream_ptr, device=f"cuda:{self.device}")

    def synchronize(self) -> None:
        _check(lib().gh_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        n = C.c_int64()
        _check(lib().gh_ctx_launch_count(self.h, C.byref(n)))
        return int(n.value)

    def set_timing(self, on: bool) -> None:
        _check(lib().gh_ctx_set_timing(self.h, int(on)))

    def reset_timing(self) -> None:
        _check(lib().gh_ctx_reset_timing(self.h))

    def set_topk_impl(self, impl: str) -> None:
        """'auto' (default), 'pick' (gather with the prune test in its loop,
        no maps), 'fused' (halo tiles, values in shared memory) or 'map'
        (map-mode gather, then k_topk_localmax on the maps)."""
        _check(lib().gh_ctx_set_topk_impl(self.h, {"auto": 0, "fused": 1, "map": 2, "pick": 3}[impl]))

    def set_debug_checks(self, on: bool) -> None:
        """Run the bounds-tested kernel builds where one exists (the top-K pick
        gather); a violation raises GridhopRuntimeError."""
        _check(lib().gh_ctx_set_debug_checks(self.h, int(on)))

    def set_direct_impl(self, impl: str) -> None:
        """'tcgen05' (default: warp-specialised 3xFP16 tensor-core pipeline),
        'tcgen05_tf32' (the same pipeline in 3xTF32), 'tcgen05_v1' (single-stage
        3xTF32 kernel), 'simt' (CUDA-core fp32) or 'tcgen05_fast' (1xFP16: one
        MMA per K step; c2 maps ~8e-5 of their maximum off, marginal against
        the 1e-4 bar, not the default)."""
        _check(lib().gh_ctx_set_direct_impl(
            self.h, {"tcgen05": 0, "simt": 1, "tcgen05_v1": 2, "tcgen05_tf32": 3,
                     "tcgen05_fast": 4}[impl]))

    def smem_peak_gbps(self) -> float:
        v = C.c_double()
        _check(lib().gh_measure_smem_peak(self.h, C.byref(v)))
        return v.value

    def kernel_time(self, name: str):
        """(total ms, launches) of kernels `name` since the last reset."""
        ms, n = C.c_double(), C.c_int64()
        _check(lib().gh_ctx_kernel_time(self.h, name.encode(), C.byref(ms), C.byref(n)))
        return ms.value, int(n.value)


class HopTable:
    """Device-resident mapping operator (HopTable, include/gridhop/interp.hpp:44-60)."""

    def __init__(self, ctx: Context, scene: Scene, handle: C.c_void_p):
        self.ctx, self.scene, self.h = ctx, scene, handle
        G, P, K, M, res = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32(), C.c_double()
        _check(lib().gh_table_info(handle, C.byref(G), C.byref(P), C.byref(K), C.byref(M),
                                   C.byref(res)))
        self.n_bins, self.n_pairs, self.k, self.n_fft = G.value, P.value, K.value, M.value
        self.max_residual = res.value

    def close(self) -> None:
        if self.h:
            _check(lib().gh_table_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def rows(self, bins):
        """(idx [n, P, K] uint32, coef [n, P, K] complex128) of the given global bins."""
        bins = np.ascontiguousarray(bins, dtype=np.int64)
        idx = np.zeros((bins.size, self.n_pairs, self.k), dtype=np.uint32)
        coef = np.zeros((bins.size, self.n_pairs, self.k), dtype=np.complex128)
        _check(lib().gh_table_rows(self.h, bins.ctypes.data, bins.size, idx.ctypes.data,
                                   coef.ctypes.data))
        return idx, coef

    def download(self):
        """(indices uint32 [G,P,K], coeffs complex128 [G,P,K]) in the reference layout."""
        n = self.n_bins * self.n_pairs * self.k
        idx = np.empty(n, dtype=np.uint32)
        coef = np.empty(2 * n, dtype=np.float64)
        _check(lib().gh_table_download(self.h, idx.ctypes.data, coef.ctypes.data))
        shape = (self.n_bins, self.n_pairs, self.k)
        return idx.reshape(shape), coef.view(np.complex128).reshape(shape)


def precompute_hop_table(ctx: Context, scene: Scene, scheme: int | None = None,
                         wrap: bool | None = None) -> HopTable:
    """precompute_hop_table (src/interp.cpp:156-223), built on the device in fp64."""
    h = C.c_void_p()
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().gh_table_build(ctx.h, C.byref(w), C.byref(g),
                                scene.scheme if scheme is None else scheme,
                                int(scene.wrap if wrap is None else wrap), C.byref(h)))
    return HopTable(ctx, scene, h)


def precompute_hop_table_shard(ctx: Context, scene: Scene, layer_lo: int, layer_hi: int,
                               scheme: int | None = None, wrap: bool | None = None,
                               halo: bool = False) -> HopTable:
    """Location-grid shard (BASELINE c5): the operator for layers [lo, hi) of
    z (3-D) / y (2-D); reported bin indices are global. halo=True builds one
    extra layer on each interior side and reports top-k peaks of [lo, hi)
    only, so per-shard top-k candidates merge exactly (distributed.merge_topk);
    maps and argmax then cover the halo layers too."""
    n_layers = scene.slab_axis_len()
    b_lo, b_hi = (max(0, layer_lo - 1), min(n_layers, layer_hi + 1)) if halo else (layer_lo, layer_hi)
    h = C.c_void_p()
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().gh_table_build_shard(ctx.h, C.byref(w), C.byref(g),
                                      scene.scheme if scheme is None else scheme,
                                      int(scene.wrap if wrap is None else wrap), b_lo, b_hi,
                                      C.byref(h)))
    t = HopTable(ctx, scene, h)
    t.bin0, _ = scene.slab_bins(b_lo, b_hi)
    t.core = (layer_lo, layer_hi)
    if halo:
        _check(lib().gh_table_set_core(h, layer_lo, layer_hi))
    return t


def upload_hop_table(ctx: Context, scene: Scene, scheme: int, idx: np.ndarray,
                     coef: np.ndarray | None) -> HopTable:
    """load_hop_table analogue: a host table in the reference layout [G][P][K]."""
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    cptr = None
    if coef is not None:
        coef = np.ascontiguousarray(coef, dtype=np.complex128)
        cptr = coef.ctypes.data
    h = C.c_void_p()
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().gh_table_upload(ctx.h, C.byref(w), C.byref(g), scheme, idx.ctypes.data, cptr,
                                 C.byref(h)))
    return HopTable(ctx, scene, h)


def _as_float_frames_mc(frames):
    torch = _torch()
    if frames.dtype != torch.complex64 or not frames.is_cuda or not frames.is_contiguous():
        raise InvalidArgument("frames must be a contiguous CUDA complex64 tensor [T, P, Mc, N]")
    return frames


def hop_map_mc(ctx: Context, table: HopTable, frames):
    """scan_planes over Mc chirps (src/hopping.cpp:59-117), K = 1 tables:
    frames complex64 [T, P, Mc, N] -> map fp32 [T, G]."""
    torch = _torch()
    frames = _as_float_frames_mc(frames)
    T, P, Mc, N = frames.shape
    if P != table.n_pairs or N != table.scene.n_samples:
        raise InvalidArgument("hop: frame shape mismatch")
    out = torch.empty((T, table.n_bins), dtype=torch.float32, device=frames.device)
    _check(lib().gh_hop_map_mc_d(ctx.h, table.h, _ptr(frames), T, Mc, _ptr(out)))
    return out


def hop_argmax_mc(ctx: Context, table: HopTable, frames):
    """hop_estimate's location stage on multi-chirp frames [T, P, Mc, N]."""
    torch = _torch()
    frames = _as_float_frames_mc(frames)
    T, P, Mc, N = frames.shape
    if P != table.n_pairs or N != table.scene.n_samples:
        raise InvalidArgument("hop: frame shape mismatch")
    idx = torch.empty(T, dtype=torch.int64, device=frames.device)
    val = torch.empty(T, dtype=torch.float32, device=frames.device)
    _check(lib().gh_hop_argmax_mc_d(ctx.h, table.h, _ptr(frames), T, Mc, _ptr(idx), _ptr(val)))
    return idx, val


def velocity(ctx: Context, scene: Scene, vgrid: VelocityGridC, frames, loc, method: str = "hop"):
    """hop_velocity / direct_velocity (src/hopping.cpp:185-236,
    src/direct.cpp:145-228) of multi-chirp frames [T, P, Mc, N] at the
    located bins loc int64 [T]: (velocity-grid index [T], value [T])."""
    torch = _torch()
    frames = _as_float_frames_mc(frames)
    T, P, Mc, N = frames.shape
    loc = loc.to(device=frames.device, dtype=torch.int64).contiguous()
    vidx = torch.empty(T, dtype=torch.int64, device=frames.device)
    vval = torch.empty(T, dtype=torch.float32, device=frames.device)
    w, g = scene.c_wave(), scene.c_grid()
    fn = lib().gh_hop_velocity_d if method == "hop" else lib().gh_direct_velocity_d
    _check(fn(ctx.h, C.byref(w), C.byref(g), C.byref(vgrid), _ptr(frames), T, Mc, _ptr(loc),
              _ptr(vidx), _ptr(vval)))
    return vidx, vval


def mrf1_write(path, frames: np.ndarray, f0: float, bandwidth: float, chirp_duration: float,
               tx_xy, rx_xy) -> None:
    """write_frames (src/frame_io.cpp:53-100): frames complex128 [T, Q, Mc, Ms]."""
    frames = np.ascontiguousarray(frames, dtype=np.complex128)
    T, Q, Mc, Ms = frames.shape
    rx = np.ascontiguousarray(rx_xy, dtype=np.float64).reshape(-1, 2)
    if rx.shape[0] != Q:
        raise InvalidArgument(f"{path}: frame/receiver count mismatch")
    h = Mrf1Header(Q, Mc, Ms, T, f0, bandwidth, chirp_duration, (C.c_double * 2)(*tx_xy))
    _check(lib().gh_mrf1_write(str(path).encode(), C.byref(h), rx.ctypes.data,
                               frames.ctypes.data if T else None))


def mrf1_read(path):
    """read_frames (src/frame_io.cpp:102-164): (header dict, rx [Q, 2],
    frames complex128 [T, Q, Mc, Ms])."""
    h = Mrf1Header()
    _check(lib().gh_mrf1_read(str(path).encode(), C.byref(h), None, 0, None, 0))
    rx = np.empty((h.n_rx, 2))
    frames = np.empty((h.n_frames, h.n_rx, h.n_chirps, h.n_samples), dtype=np.complex128)
    _check(lib().gh_mrf1_read(str(path).encode(), C.byref(h), rx.ctypes.data, h.n_rx,
                              frames.ctypes.data, frames.size))
    hdr = {f: getattr(h, f) for f, _ in Mrf1Header._fields_ if f != "tx"}
    hdr["tx"] = (h.tx[0], h.tx[1])
    return hdr, rx, frames


def indirect_argmin(ctx: Context, scene: Scene, frames):
    """Indirect pipeline location stage (src/indirect.cpp:10-83, Mc = 1):
    (r_hat fp64 [T, P], bin int64 [T], residual fp64 [T])."""
    torch = _torch()
    frames = _scene_frames(scene, frames)
    T = frames.shape[0]
    dev = frames.device
    rhat = torch.empty((T, scene.n_pairs), dtype=torch.float64, device=dev)
    idx = torch.empty(T, dtype=torch.int64, device=dev)
    res = torch.empty(T, dtype=torch.float64, device=dev)
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().gh_indirect_argmin_d(ctx.h, C.byref(w), C.byref(g), _ptr(frames), T, _ptr(rhat),
                                      _ptr(idx), _ptr(res)))
    return rhat, idx, res


def multilaterate(ctx: Context, scene: Scene, rhat):
    """multilaterate_location (src/indirect.cpp:58-83) on device range
    estimates rhat fp64 [T, P]: (bin int64 [T], residual fp64 [T])."""
    torch = _torch()
    rhat = rhat.contiguous()
    T = rhat.shape[0]
    idx = torch.empty(T, dtype=torch.int64, device=rhat.device)
    res = torch.empty(T, dtype=torch.float64, device=rhat.device)
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().gh_multilaterate_d(ctx.h, C.byref(w), C.byref(g), _ptr(rhat), T, _ptr(idx),
                                    _ptr(res)))
    return idx, res


def scene_hash(n_chirps: int, n_samples: int, f0: float, bandwidth: float,
               chirp_duration: float, tx_xy, rx_xy) -> int:
    """scene_hash (src/model.cpp:135-166) of a single-TX 2-D geometry."""
    tx = np.ascontiguousarray(tx_xy, dtype=np.float64).reshape(2)
    rx = np.ascontiguousarray(rx_xy, dtype=np.float64).reshape(-1, 2)
    return int(lib().gh_scene_hash(rx.shape[0], n_chirps, n_samples, f0, bandwidth, chirp_duration,
                                   tx.ctypes.data, rx.ctypes.data))


def ght1_write(path: str, idx: np.ndarray, coef: np.ndarray, os_range: int, n_samples: int,
               scene_hash: int, max_residual: float = 0.0) -> None:
    """save_hop_table (src/interp.cpp:293-317) of a host table [G][P][K]."""
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    coef = np.ascontiguousarray(coef, dtype=np.complex128)
    G, P, K = idx.shape
    h = Ght1Header(P, G, K, os_range, n_samples, scene_hash, max_residual)
    _check(lib().gh_ght1_write(str(path).encode(), C.byref(h), idx.ctypes.data, coef.ctypes.data))


def ght1_read(path: str):
    """load_hop_table's parser (src/interp.cpp:319-380): (header dict, idx
    uint32 [G,P,K], coeffs complex128 [G,P,K])."""
    h = Ght1Header()
    _check(lib().gh_ght1_read(str(path).encode(), C.byref(h), None, None, 0))
    shape = (h.n_bins, h.n_pairs, h.k)
    n = h.n_bins * h.n_pairs * h.k
    idx = np.empty(n, dtype=np.uint32)
    coef = np.empty(n, dtype=np.complex128)
    _check(lib().gh_ght1_read(str(path).encode(), C.byref(h), idx.ctypes.data, coef.ctypes.data, n))
    hdr = {f: getattr(h, f) for f, _ in Ght1Header._fields_}
    return hdr, idx.reshape(shape), coef.reshape(shape)


def table_save(table: HopTable, path: str, scene_hash: int) -> None:
    """save_hop_table of a device table (GHT1)."""
    _check(lib().gh_table_save(table.h, str(path).encode(), scene_hash))


def table_load(ctx: Context, path: str, scene: Scene, scene_hash: int) -> HopTable:
    """load_hop_table: validated against `scene` ("stale hop table"), uploaded."""
    h = C.c_void_p()
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().gh_table_load(ctx.h, str(path).encode(), C.byref(w), C.byref(g), scene_hash,
                               C.byref(h)))
    return HopTable(ctx, scene, h)


def _as_float_frames(frames, n_pairs: int | None = None, n_samples: int | None = None):
    """Device frames complex64 [T, P, N]; with (n_pairs, n_samples) given the
    per-trial shape must match ("hop: frame shape mismatch",
    src/hopping.cpp:251) — the C ABI takes only T and reads P*N per trial."""
    torch = _torch()
    if frames.dtype != torch.complex64 or not frames.is_cuda or not frames.is_contiguous():
        raise InvalidArgument("frames must be a contiguous CUDA complex64 tensor [T, P, N]")
    if frames.dim() != 3:
        raise InvalidArgument("hop: frame shape mismatch")
    if n_pairs is not None and (frames.shape[1] != n_pairs or frames.shape[2] != n_samples):
        raise InvalidArgument("hop: frame shape mismatch")
    return frames


def _table_frames(table: "HopTable", frames):
    return _as_float_frames(frames, table.n_pairs, table.scene.n_samples)


def _scene_frames(scene: Scene, frames):
    return _as_float_frames(frames, scene.n_pairs, scene.n_samples)


def _as_maps(scene: Scene, maps):
    torch = _torch()
    if (maps.dtype != torch.float32 or not maps.is_cuda or maps.dim() != 2
            or maps.shape[1] != scene.n_bins):
        raise InvalidArgument("top-k: maps must be a CUDA float32 tensor [T, n_bins]")
    return maps.contiguous()


def synthesize(ctx: Context, scene: Scene, trial0: int, n_trials: int, snr_db=None,
               wrap: bool | None = None):
    """synthesize_frame + add_noise (src/synth.cpp:15-49) for a batch of trials.

    Returns (frames complex64 [T, P, N], truth float64 [T, K, 3]) on the device."""
    torch = _torch()
    dev = f"cuda:{ctx.device}"
    frames = torch.empty((n_trials, scene.n_pairs, scene.n_samples), dtype=torch.complex64, device=dev)
    truth = torch.empty((n_trials, scene.n_targets, 3), dtype=torch.float64, device=dev)
    w, camp = scene.c_wave(), scene.c_campaign(snr_db)
    _check(lib().gh_synth_d(ctx.h, C.byref(w), C.byref(camp), trial0, n_trials,
                            int(scene.wrap if wrap is None else wrap), _ptr(frames), _ptr(truth)))
    return frames, truth


def fast_time_spectra(ctx: Context, frames, os_range: int):
    """fast_time_spectra (src/hopping.cpp:121-129): [T, P, N] -> [T, P, os*N]."""
    torch = _torch()
    frames = _as_float_frames(frames)
    T, P, N = frames.shape
    out = torch.empty((T, P, N * os_range), dtype=torch.complex64, device=frames.device)
    _check(lib().gh_spectra_d(ctx.h, _ptr(frames), T, P, N, os_range, _ptr(out)))
    return out


def hop_decision_map(ctx: Context, table: HopTable, frames, combine: int = POWER):
    """hop_decision_map (src/hopping.cpp:179-183) for T trials: fp32 [T, G]."""
    torch = _torch()
    frames = _table_frames(table, frames)
    out = torch.empty((frames.shape[0], table.n_bins), dtype=torch.float32, device=frames.device)
    _check(lib().gh_hop_map_d(ctx.h, table.h, _ptr(frames), frames.shape[0], combine, _ptr(out)))
    return out


def hop_argmax(ctx: Context, table: HopTable, frames, combine: int = POWER):
    """hop_estimate location stage (src/hopping.cpp:238-267) batched: (idx, value)."""
    torch = _torch()
    frames = _table_frames(table, frames)
    T = frames.shape[0]
    idx = torch.empty(T, dtype=torch.int64, device=frames.device)
    val = torch.empty(T, dtype=torch.float32, device=frames.device)
    _check(lib().gh_hop_argmax_d(ctx.h, table.h, _ptr(frames), T, combine, _ptr(idx), _ptr(val)))
    return idx, val


def hop_estimate(ctx: Context, table: HopTable, frames: np.ndarray, combine: int = POWER,
                 out_idx: np.ndarray | None = None, out_val: np.ndarray | None = None):
    """Host-buffer hop estimate: complex128 frames [T, P, N] -> (idx int64, value f64)."""
    frames = np.ascontiguousarray(frames, dtype=np.complex128)
    T = frames.shape[0]
    if frames.ndim != 3 or frames.shape[1] != table.n_pairs or frames.shape[2] != table.scene.n_samples:
        raise InvalidArgument("hop: frame shape mismatch")
    idx = np.empty(T, dtype=np.int64) if out_idx is None else out_idx
    val = np.empty(T, dtype=np.float64) if out_val is None else out_val
    _check(lib().gh_hop_estimate(ctx.h, table.h, frames.ctypes.data, T, combine,
                                 idx.ctypes.data, val.ctypes.data))
    return idx, val


def hop_estimate_ptr(ctx: Context, table: HopTable, frames_ptr: int, n_trials: int,
                     combine: int, idx_ptr: int, val_ptr: int) -> None:
    """Raw-pointer form (pinned host buffers from the bench)."""
    _check(lib().gh_hop_estimate(ctx.h, table.h, frames_ptr, n_trials, combine, idx_ptr, val_ptr))


def hop_estimate_topk(ctx: Context, table: HopTable, frames: np.ndarray, k: int,
                      combine: int = POWER):
    """Host-buffer multi-target estimate: complex128 frames [T, P, N] ->
    (idx int64 [T, k], value f64 [T, k]), top-k local maxima of each map."""
    frames = np.ascontiguousarray(frames, dtype=np.complex128)
    if frames.ndim != 3 or frames.shape[1] != table.n_pairs or frames.shape[2] != table.scene.n_samples:
        raise InvalidArgument("hop: frame shape mismatch")
    T = frames.shape[0]
    idx = np.empty((T, k), dtype=np.int64)
    val = np.empty((T, k), dtype=np.float64)
    _check(lib().gh_hop_estimate_topk(ctx.h, table.h, frames.ctypes.data, T, combine, k,
                                      idx.ctypes.data, val.ctypes.data))
    return idx, val


def hop_estimate_topk_ptr(ctx: Context, table: HopTable, frames_ptr: int, n_trials: int,
                          combine: int, k: int, idx_ptr: int, val_ptr: int) -> None:
    """Raw-pointer form (pinned host buffers from the bench)."""
    _check(lib().gh_hop_estimate_topk(ctx.h, table.h, frames_ptr, n_trials, combine, k, idx_ptr,
                                      val_ptr))


def campaign_hop(ctx: Context, table: HopTable, scene: Scene, trial0: int, n_trials: int,
                 combine: int = POWER, snr_db=None, out=None):
    """One Monte-Carlo step of the hop arm (src/montecarlo.cpp:140-175):
    synthesis fused into the FFT, gather, argmax. Returns (idx, value)."""
    torch = _torch()
    dev = f"cuda:{ctx.device}"
    if out is None:
        idx = torch.empty(n_trials, dtype=torch.int64, device=dev)
        val = torch.empty(n_trials, dtype=torch.float32, device=dev)
    else:
        idx, val = out
    camp = scene.c_campaign(snr_db)
    _check(lib().gh_campaign_hop_d(ctx.h, table.h, C.byref(camp), trial0, n_trials, combine,
                                   _ptr(idx), _ptr(val)))
    return idx, val


def hop_topk(ctx: Context, table: HopTable, frames, k: int, combine: int = POWER):
    """Top-k local maxima of each trial's hop map (BASELINE c3): (idx [T,k], val [T,k])."""
    torch = _torch()
    frames = _table_frames(table, frames)
    T = frames.shape[0]
    idx = torch.empty((T, k), dtype=torch.int64, device=frames.device)
    val = torch.empty((T, k), dtype=torch.float32, device=frames.device)
    _check(lib().gh_hop_topk_d(ctx.h, table.h, _ptr(frames), T, combine, k, _ptr(idx), _ptr(val)))
    return idx, val


def campaign_hop_topk(ctx: Context, table: HopTable, scene: Scene, trial0: int, n_trials: int,
                      k: int, combine: int = POWER, snr_db=None):
    torch = _torch()
    dev = f"cuda:{ctx.device}"
    idx = torch.empty((n_trials, k), dtype=torch.int64, device=dev)
    val = torch.empty((n_trials, k), dtype=torch.float32, device=dev)
    camp = scene.c_campaign(snr_db)
    _check(lib().gh_campaign_hop_topk_d(ctx.h, table.h, C.byref(camp), trial0, n_trials, combine, k,
                                        _ptr(idx), _ptr(val)))
    return idx, val


def topk_local_max(ctx: Context, scene: Scene, maps, k: int):
    """Top-k local maxima of caller maps fp32 [T, G] on the device."""
    torch = _torch()
    maps = _as_maps(scene, maps)
    T = maps.shape[0]
    idx = torch.empty((T, k), dtype=torch.int64, device=maps.device)
    val = torch.empty((T, k), dtype=torch.float32, device=maps.device)
    g = scene.c_grid()
    _check(lib().gh_topk_local_max_d(ctx.h, C.byref(g), _ptr(maps), T, k, _ptr(idx),
                                     _ptr(val)))
    return idx, val


def location_decision_map(ctx: Context, scene: Scene, frames, combine: int = POWER):
    """location_decision_map (src/direct.cpp:90-144) for T trials: fp32 [T, G]."""
    torch = _torch()
    frames = _scene_frames(scene, frames)
    out = torch.empty((frames.shape[0], scene.n_bins), dtype=torch.float32, device=frames.device)
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().gh_direct_map_d(ctx.h, C.byref(w), C.byref(g), _ptr(frames), frames.shape[0],
                                 combine, _ptr(out)))
    return out


def direct_argmax(ctx: Context, scene: Scene, frames, combine: int = POWER):
    """direct_estimate location stage (src/direct.cpp:230-239) batched: (idx, value)."""
    torch = _torch()
    frames = _scene_frames(scene, frames)
    T = frames.shape[0]
    idx = torch.empty(T, dtype=torch.int64, device=frames.device)
    val = torch.empty(T, dtype=torch.float32, device=frames.device)
    w, g = scene.c_wave(), scene.c_grid()
    _check(lib().gh_direct_argmax_d(ctx.h, C.byref(w), C.byref(g), _ptr(frames), T, combine,
                                    _ptr(idx), _ptr(val)))
    return idx, val


def argmax_index(values) -> int:
    """argmax_index (src/direct.cpp:55-62): first strict maximum."""
    v = np.asarray(values)
    if v.size == 0:
        raise InvalidArgument("argmax of empty scan")
    return int(np.argmax(v))  # numpy returns the first occurrence of the max


# ---------------------------------------------------------------- multi-GPU + campaigns
def comm_unique_id() -> bytes:
    """ncclGetUniqueId on this rank (rank 0), to broadcast to the others."""
    buf = (C.c_uint8 * 128)()
    _check(lib().gh_comm_unique_id(buf))
    return bytes(buf)


class Comm:
    """gh_comm: one NCCL communicator rank on `ctx`'s device (one process
    per GPU). `uid` comes from comm_unique_id() on rank 0."""

    def __init__(self, ctx: Context, uid: bytes, n_ranks: int, rank: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(lib().gh_comm_init(ctx.h, buf, n_ranks, rank, C.byref(h)))
        self.h, self.n_ranks, self.rank = h, n_ranks, rank

    @classmethod
    def from_torch_distributed(cls, ctx: Context) -> "Comm":
        """Rank 0's id broadcast over the initialised torch.distributed group."""
        import torch.distributed as dist
        obj = [comm_unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(ctx, obj[0], dist.get_world_size(), dist.get_rank())

    def close(self) -> None:
        if self.h:
            _check(lib().gh_comm_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def campaign_run(ctx: Context, scene: Scene, n_trials: int | None = None, algorithms=("hop",),
                 snr_db=None, densities=None, thresholds=None, topk: int | None = None,
                 comm: Comm | None = None, batch: int = 0, trial_csv=None, summary_csv=None,
                 scheme: int | None = None, wrap: bool | None = None, combine: int = POWER):
    """run_monte_carlo (src/montecarlo.cpp:99-179) on the device: every
    (density, SNR, algorithm) cell over n_trials trials (sharded over
    `comm`'s ranks), statistics on the device, one NCCL all-reduce per cell.
    snr_db: None = the scene's SNR model (one cell), else a list (NaN =
    noiseless). Returns one dict per cell (record order density, SNR,
    algorithm) with hit ratios per threshold, RMSE, half-resolution hits and
    the device times."""
    algos = [ALGO_IDS[a] if isinstance(a, str) else int(a) for a in algorithms]
    alg_arr = (C.c_int32 * len(algos))(*algos)
    d = CampaignDesc()
    d.wave = scene.c_wave()
    d.grid = scene.c_grid()
    d.scene = scene.c_campaign()
    d.scheme = scene.scheme if scheme is None else scheme
    d.wrap = int(scene.wrap if wrap is None else wrap)
    d.combine = combine
    d.n_algorithms = len(algos)
    d.algorithms = alg_arr
    keep = [alg_arr]
    if snr_db is not None:
        arr = (C.c_double * len(snr_db))(*[float(x) for x in snr_db])
        keep.append(arr)
        d.n_snr, d.snr_db = len(snr_db), arr
    if densities is not None:
        arr = (C.c_double * len(densities))(*[float(x) for x in densities])
        keep.append(arr)
        d.n_density, d.density = len(densities), arr
    if thresholds is not None:
        arr = (C.c_double * len(thresholds))(*[float(x) for x in thresholds])
        keep.append(arr)
        d.n_thresholds, d.thresholds_m = len(thresholds), arr
    d.n_trials = int(scene.trials if n_trials is None else n_trials)
    d.topk = int(topk or scene.topk)
    d.batch = int(batch)
    d.trial_csv = str(trial_csv).encode() if trial_csv else None
    d.summary_csv = str(summary_csv).encode() if summary_csv else None
    n_cells = max(1, len(densities or [1])) * max(1, len(snr_db or [0])) * len(algos)
    out = (CellStats * n_cells)()
    got = C.c_int32()
    _check(lib().gh_campaign_run(ctx.h, comm.h if comm else None, C.byref(d), out, n_cells,
                                 C.byref(got)))
    names = {v: k for k, v in ALGO_IDS.items()}
    cells = []
    for cs in out[:got.value]:
        nth = cs.n_thresholds
        cells.append({
            "algorithm": names[cs.algorithm], "density": cs.density, "snr_db": cs.snr_db,
            "trials": cs.trials, "estimates": cs.estimates,
            "thresholds_m": list(cs.thresholds_m[:nth]), "hits": list(cs.hits[:nth]),
            "hit_ratio": list(cs.hit_ratio[:nth]), "hits_half_res": cs.hits_half_res,
            "sq_err_sum": cs.sq_err_sum, "err_sum": cs.err_sum, "rmse_m": cs.rmse_m,
            "online_ms": cs.online_ms, "offline_ms": cs.offline_ms,
            "mean_online_ns": cs.mean_online_ns})
    return cells
