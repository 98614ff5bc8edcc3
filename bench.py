#!/usr/bin/env python
"""Benchmark of the grid-hopping hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c3]

Default workload: BASELINE c3, the largest configuration that fits one GPU
(the metric is not quoted on a config): 100,000 Monte-Carlo trials per GPU,
10^6 location bins x 16 TX-RX pairs, N = 1024, M = 4096, 5 targets, top-5
local-maximum peak pick. One step = one pass of the hop pipeline over the
step's trials: zero-padded range FFT -> gather-accumulate through the mapping
operator -> per-trial top-5 local maxima. Inputs (complex64 beat signals) are
resident in HBM before timing (`value`); `e2e` runs the reference-facing host
call gh_hop_estimate_topk on pinned complex128 frames with the copies inside
the timed region. `--config c1|c2|c4` run the other trial-sharded configs
(argmax), `--config c5` the location-grid-sharded 3-D config.

Multi-GPU: one process per GPU (`--gpus N` re-launches itself under
torch.distributed.run when not already a rank); each rank owns its own block
of trials (weak scaling, no data-path collective); the step time is the max
over ranks.

The reference arm (`--impl reference`) times the CPU restatement of the
reference pipeline (oracle/, fp64, parallel_for over trials on every host
core) on a bounded sample of the same workload; the reference itself cannot
be built (Eigen3/FFTW3 absent).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "location-bin x pair correlations/s (grid hopping)"
UNIT = "bin*pair correlations/s"


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "fallback": True}


# gather instantiation per BASELINE config: its ncu --set full capture in
# profiles/ supplies roofline.traffic (DRAM read + write per launch)
GATHER_KERNEL = {"c1": "k_gather<16, 0, 0, 0, 3, 1", "c2": "k_gather<16, 0, 0, 0, 3, 1",
                 "c3": "k_gather_pick<16, 4", "c4": "k_gather<16, 1, 0, 0, 16, 4"}
GATHER_LABEL = {"c1": "k_gather (fused argmax)", "c2": "k_gather (fused argmax)",
                "c3": "k_gather_pick (gather with the top-K prune test in its loop, no maps)",
                "c4": "k_gather (K = 3, fused argmax)"}


def ncu_traffic(config: str, trials: int):
    """DRAM bytes per launch of the config's gather kernel from the newest
    committed ncu --set full summary (profiles/r*_kernels_ncu_full.json),
    scaled to `trials` (captures run tools/prof_step.py at their own trial
    count, recorded in profiles/README.md); None when absent."""
    want = GATHER_KERNEL.get(config)
    files = sorted((ROOT / "profiles").glob("r*_kernels_ncu_full.json"))
    if not want or not files:
        return None
    data = json.loads(files[-1].read_text())
    for rep, kernels in data.items():
        for k in kernels:
            if want in k.get("kernel", "") and k.get("dram_read_bytes") is not None:
                t0 = next((n for pre, n in PROFILE_TRIALS.items() if rep.startswith(pre + "_r")),
                          None)
                if not t0:
                    continue
                return (k["dram_read_bytes"] + k.get("dram_write_bytes", 0.0)) * trials / t0
    return None


# trials per launch of each committed capture (tools/evidence*.sh), by report prefix
PROFILE_TRIALS = {"prof_hop": 10000, "prof_c3": 2048, "prof_c3fused": 2048, "prof_c3pick": 9472,
                  "prof_c4": 2000, "prof_c5": 64, "prof_direct": 1024}


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled through NVML every
    ~1 ms during the timed region (the same counters nvidia-smi reads; the
    timed region is only milliseconds long)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, device: int):
        self.device = device
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self.stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            time.sleep(0.005)
        except Exception:
            self.ok = False
        return self

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                clk = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((clk, rs))
            except Exception:
                pass
            time.sleep(0.001)

    def __exit__(self, *exc):
        self.stop.set()
        if self.ok:
            self.t.join(timeout=2)

    def summary(self) -> dict:
        sm = [c for c, _ in self.samples]
        reasons = set()
        for _, rs in self.samples:
            for bit, name in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm), "source": "NVML, 1 ms poll"}


def tensor_peak_tflops(device: int, dtype: str) -> float:
    """Dense tensor-core peak measured in-run with cuBLAS 8192^3 GEMMs, best of
    6: dtype "fp16" (the pipe kind::f16 MMAs use; MEASURED_PEAKS.json's bf16
    figure is its sibling) or "tf32" (fp32 inputs on the TF32 tensor cores)."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        dt = torch.float16 if dtype == "fp16" else torch.float32
        a = torch.randn(n, n, device=f"cuda:{device}", dtype=dt)
        b = torch.randn(n, n, device=f"cuda:{device}", dtype=dt)
        best = float("inf")
        for _ in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _oracle_campaign(O, sc, oi, oc, trial0, n, nthr):
    if sc.topk > 1:
        return O.campaign_hop_topk(sc, oi, oc, trial0, n, sc.topk, threads=nthr)
    return O.campaign_hop(sc, oi, oc, trial0, n, threads=nthr)


def _pick_label(sc) -> str:
    return f"top-{sc.topk} local maxima" if sc.topk > 1 else "argmax"


def cpu_baseline(sc, oi, oc, target_s: float = 20.0, kind: str = "port") -> dict:
    """The oracle's per-trial pipeline (synth -> FFT -> hop scan in 1024-bin
    chunks -> argmax / top-k) with parallel_for over trials on all host cores,
    timed on the first trials of the campaign (a bounded sample)."""
    from oracle import oracle as O
    nthr = O.nthreads()
    n = max(nthr, 8)
    t0 = time.perf_counter()
    _oracle_campaign(O, sc, oi, oc, 0, n, nthr)
    dt = time.perf_counter() - t0
    n2 = int(max(nthr, min(2_000_000, n * target_s / max(dt, 1e-3))))
    t0 = time.perf_counter()
    _oracle_campaign(O, sc, oi, oc, 0, n2, nthr)
    dt = time.perf_counter() - t0
    units = n2 * sc.units_per_trial()
    return {"value": units / dt, "unit": UNIT, "cores": nthr, "kind": kind,
            "trials_per_s": n2 / dt,
            "sample": f"first {n2} trials of the {sc.name} campaign ({_pick_label(sc)}), "
                      f"{dt:.1f} s, fp64, {nthr} threads; value = their bin*pair rate"}


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU pipeline (oracle port) on this
    arm's config, rank 0 only (other ranks exit without work)."""
    if rank != 0:
        return
    from paper_2307_16550_b200 import scene as S
    from oracle import oracle as O
    sc = S.baseline(args.config)
    oi, oc, _ = O.build_table(sc)
    nthr = O.nthreads()
    # bounded sample per step so that warmup + steps end within minutes
    t0 = time.perf_counter()
    _oracle_campaign(O, sc, oi, oc, 0, nthr, nthr)
    per_trial = (time.perf_counter() - t0) / nthr
    budget = args.ref_seconds / max(1, args.steps + args.warmup)
    per_step = int(max(nthr, min(sc.trials, args.ref_trials or 10**9, budget / max(per_trial, 1e-9))))
    per_step = max(nthr, per_step // nthr * nthr)
    for _ in range(args.warmup):
        _oracle_campaign(O, sc, oi, oc, 0, max(nthr, per_step // 4), nthr)
    t0 = time.perf_counter()
    for k in range(args.steps):
        _oracle_campaign(O, sc, oi, oc, k * per_step, per_step, nthr)
    dt = (time.perf_counter() - t0) / args.steps
    value = per_step * sc.units_per_trial() / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter-based RNG, seed 20260816)",
        "config": {"workload": f"{sc.name}: {per_step} trials/step sample of {sc.trials}, "
                               f"{sc.n_bins} bins x {sc.n_pairs} pairs, N={sc.n_samples}, "
                               f"M={sc.n_fft}, {S.SCHEME_NAMES[sc.scheme]} (K={sc.k}), "
                               f"{_pick_label(sc)}",
                   "bins": sc.n_bins, "pairs": sc.n_pairs, "n_samples": sc.n_samples,
                   "n_fft": sc.n_fft, "scheme": S.SCHEME_NAMES[sc.scheme], "topk": sc.topk},
        "trials_per_s": per_step / dt,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthr, "kind": "port",
                         "sample": f"{per_step} trials per step (trials k*{per_step}.. of the "
                                   f"campaign), fp64, {nthr} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference (Eigen3/FFTW3) not buildable here; fp64 oracle port of its "
                "pipeline, parallel_for over trials on all host cores",
    }
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import torch
    import paper_2307_16550_b200 as gh
    from paper_2307_16550_b200 import scene as S

    dist = world > 1
    if dist:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    sc = S.baseline(args.config)
    T = args.trials or sc.trials
    G, P, N = sc.n_bins, sc.n_pairs, sc.n_samples
    dev = f"cuda:{local}"
    ctx = gh.Context(local)
    stream = ctx.torch_stream()
    table = gh.precompute_hop_table(ctx, sc)
    trial0 = rank * T  # weak scaling: every rank owns its own trials
    frames, _ = gh.synthesize(ctx, sc, trial0, T)
    ctx.synchronize()
    # L2 is 126 MB: c1/c2 frames (61 MB) + spectra (123 MB) would partly stay
    # resident, so L2 is flushed between timed steps (outside the events);
    # the c3/c4 inputs (13 GB / 5 GB) exceed it anyway
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def barrier():
        if dist:
            tdist.barrier()
        torch.cuda.synchronize()

    topk = sc.topk if sc.topk > 1 else 0  # BASELINE c3: top-K local-maximum pick

    def step():
        if topk:
            return gh.hop_topk(ctx, table, frames, topk)
        return gh.hop_argmax(ctx, table, frames)

    for _ in range(max(3, args.warmup)):
        step()
    ctx.synchronize()
    smem_peak = ctx.smem_peak_gbps()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    # The headline loop carries only the step events: per-kernel event pairs
    # cost ~5 % of a c2 step, so the kernel times for the roofline come from
    # a second pass of the same K steps (same L2 flush) with them enabled.
    launches0 = ctx.launches
    barrier()
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                flush.zero_()
                evs[k][0].record(stream)
                idx, val = step()
                evs[k][1].record(stream)
        ctx.synchronize()
        t_wall = time.perf_counter() - t_wall
    barrier()
    launches = ctx.launches - launches0
    ms_steps = [a.elapsed_time(b) for a, b in evs]
    ms = sum(ms_steps) / len(ms_steps)
    ctx.reset_timing()
    ctx.set_timing(not args.no_kernel_timing)
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            flush.zero_()
            step()
    ctx.synchronize()
    ctx.set_timing(False)
    kern = {name: ctx.kernel_time(name) for name in ("fft", "gather", "decode", "topk", "merge")}
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    units_step = T * G * P * world
    value = units_step / (ms * 1e-3)
    clocks = clk.summary()

    # ---- e2e: reference-facing host call on pinned complex128 frames (the
    # reference's FrameSet element type), H2D + D2H inside the timed region
    kk = max(topk, 1)
    fr_host = torch.empty((T, P, N), dtype=torch.complex128, pin_memory=True)
    for a0 in range(0, T, 8192):
        fr_host[a0:a0 + 8192].copy_(frames[a0:a0 + 8192].cpu())
    idx_h = torch.empty((T, kk), dtype=torch.int64, pin_memory=True)
    val_h = torch.empty((T, kk), dtype=torch.float64, pin_memory=True)

    def e2e_step():
        if topk:
            gh.api.hop_estimate_topk_ptr(ctx, table, fr_host.data_ptr(), T, S.POWER, topk,
                                         idx_h.data_ptr(), val_h.data_ptr())
        else:
            gh.api.hop_estimate_ptr(ctx, table, fr_host.data_ptr(), T, S.POWER, idx_h.data_ptr(),
                                    val_h.data_ptr())

    for _ in range(2):
        e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = (time.perf_counter() - t0) / args.steps
    # this box's raw pinned H2D rate (a 1 GB copy), the bound e2e runs
    # against when the frames cross PCIe as complex128
    n_probe = min(T, max(1, (1 << 30) // (P * N * 16)))
    dst = torch.empty((n_probe, P, N), dtype=fr_host.dtype, device=dev)
    dst.copy_(fr_host[:n_probe], non_blocking=True)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for _ in range(3):
        dst.copy_(fr_host[:n_probe], non_blocking=True)
    torch.cuda.synchronize()
    h2d_gbs = 3 * dst.numel() * dst.element_size() / (time.perf_counter() - h0) / 1e9
    del dst
    if dist:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # same answers through both entry points
    assert np.array_equal(idx_h.numpy().reshape(T, -1), idx.cpu().numpy().reshape(T, -1))
    del fr_host

    # ---- Monte-Carlo campaign step (synthesis fused into the FFT)
    def camp_step():
        if topk:
            return gh.campaign_hop_topk(ctx, table, sc, trial0, T, topk)
        return gh.campaign_hop(ctx, table, sc, trial0, T)

    for _ in range(2):
        camp_step()
    ctx.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for k in range(args.steps):
            camp_step()
        e1.record(stream)
    ctx.synchronize()
    camp_ms = e0.elapsed_time(e1) / args.steps

    # ---- direct method (BASELINE c2 "run both ways"): tcgen05 3xFP16
    direct = None
    if not args.no_direct and sc.name in ("c1", "c2"):
        for _ in range(2):
            gh.direct_argmax(ctx, sc, frames)
        ctx.synchronize()
        ctx.reset_timing()
        ctx.set_timing(True)
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            d0.record(stream)
            for _ in range(args.direct_steps):
                didx, _ = gh.direct_argmax(ctx, sc, frames)
            d1.record(stream)
        ctx.synchronize()
        ctx.set_timing(False)
        dk_ms, dk_n = ctx.kernel_time("direct_umma")
        dstep_ms = d0.elapsed_time(d1) / args.direct_steps
        flops = 8.0 * N * G * P * T  # algorithmic: one complex MAC = 8 flops
        f16_peak = tensor_peak_tflops(local, "fp16")
        tf32_peak = tensor_peak_tflops(local, "tf32")
        agree = float(np.mean(didx.cpu().numpy() == idx.cpu().numpy()))
        kern_ms = dk_ms / max(dk_n, 1)
        alg = flops / (kern_ms * 1e-3) / 1e12
        direct = {"ms_per_step": dstep_ms, "kernel_ms": kern_ms,
                  "trials_per_s": T * world / (dstep_ms * 1e-3),
                  "value": units_step / (dstep_ms * 1e-3),
                  "tflops_algorithmic": alg,
                  "roofline": {"bound": "tensor", "unit": "TFLOP/s", "peak": f16_peak,
                               "peak_source": "torch.matmul fp16 8192^3 (cuBLAS), measured in-run: "
                                              "the kind::f16 tensor pipe the kernel uses",
                               "achieved": alg, "frac": alg / f16_peak,
                               "executed_mma_factor": 3,
                               "executed_frac": 3 * alg / f16_peak,
                               "tf32_peak": tf32_peak,
                               "note": "3xFP16 issues 3 MMAs per algorithmic MAC; achieved counts "
                                       "the algorithmic 8NGP flops only"},
                  "hop_direct_argmax_agreement": agree,
                  "api": "gh_direct_argmax_d (tcgen05 kind::f16, 3xFP16)"}
        # the 1xFP16 fast mode (one MMA per K step): marginal against the parity
        # bar (c2 maps ~8e-5 of their maximum off), reported beside the default
        ctx.set_direct_impl("tcgen05_fast")
        try:
            for _ in range(2):
                gh.direct_argmax(ctx, sc, frames)
            ctx.synchronize()
            ctx.reset_timing()
            ctx.set_timing(True)
            for _ in range(args.direct_steps):
                fidx, _ = gh.direct_argmax(ctx, sc, frames)
            ctx.synchronize()
            ctx.set_timing(False)
            fk_ms, fk_n = ctx.kernel_time("direct_umma")
            fk = fk_ms / max(fk_n, 1)
            falg = flops / (fk * 1e-3) / 1e12
            direct["fast_1xfp16"] = {
                "kernel_ms": fk, "tflops_algorithmic": falg, "frac_of_fp16_peak": falg / f16_peak,
                "argmax_agreement_with_3xfp16": float(np.mean(fidx.cpu().numpy()
                                                              == didx.cpu().numpy())),
                "note": "gh_ctx_set_direct_impl(4): fp16 operands, c2 maps ~8e-5 of their maximum "
                        "off (marginal against the 1e-4 bar), not the default; bounded in "
                        "tests/test_gpu_parity.py; the steering generation, not the tensor pipe, "
                        "then bounds the kernel"}
        finally:
            ctx.set_direct_impl("tcgen05")

    # ---- indirect pipeline location stage (range peaks + multilateration,
    # src/indirect.cpp:10-83): the reference's third comparison arm
    indirect = None
    if not args.no_direct and sc.name in ("c1", "c2"):
        for _ in range(2):
            gh.indirect_argmin(ctx, sc, frames)
        ctx.synchronize()
        ctx.reset_timing()
        ctx.set_timing(True)
        i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            i0.record(stream)
            for _ in range(args.direct_steps):
                _, iidx, _ = gh.indirect_argmin(ctx, sc, frames)
            i1.record(stream)
        ctx.synchronize()
        ctx.set_timing(False)
        ims = i0.elapsed_time(i1) / args.direct_steps
        ml_ms, ml_n = ctx.kernel_time("multilaterate")
        indirect = {"ms_per_step": ims, "trials_per_s": T * world / (ims * 1e-3),
                    "multilaterate_ms": ml_ms / max(ml_n, 1),
                    "hop_indirect_argmax_agreement": float(np.mean(iidx.cpu().numpy()
                                                                   == idx.cpu().numpy())),
                    "api": "gh_indirect_argmin_d (FFT, range peaks, fp64 multilateration)"}

    if rank != 0:
        if dist:
            tdist.destroy_process_group()
        return
    pk = peaks()
    g_ms, g_n = kern["gather"]
    g_avg = g_ms / args.steps  # per step (top-K steps run the gather once per trial chunk)
    # per launch (top-K steps may launch the gather once per trial chunk)
    g_launches = max(1, g_n // args.steps)
    t_launch = T / g_launches
    g_launch_ms = max(g_avg / g_launches, 1e-9)  # (no kernel timing: diagnostic runs only)
    # shared-memory bytes gathered per unit: fp32 power (K = 1) or three
    # complex64 spectrum values (K = 3)
    lsu_bytes = t_launch * G * P * (4.0 if sc.k == 1 else 24.0)
    achieved = lsu_bytes / (g_launch_ms * 1e-3) / 1e9
    # staged spectra (fp32 power, or complex64 for K = 3) + table rows
    hbm_bytes = (t_launch * P * sc.n_fft * (4.0 if sc.k == 1 else 8.0) + G * 8
                 + (G * P * 24 if sc.k == 3 else 0))
    kernels_ms = {k: v[0] / args.steps for k, v in kern.items() if v[1]}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": f"synthetic (counter-based RNG, seed 20260816), {sc.name} scene",
        "config": {"workload": f"{sc.name}: {T} trials/GPU, {G} bins x {P} pairs, N={N}, "
                               f"M={sc.n_fft}, {S.SCHEME_NAMES[sc.scheme]} (K={sc.k}), power sum, "
                               f"{'wrap mode' if sc.wrap else 'reference window check'}, "
                               f"{_pick_label(sc)}",
                   "trials_per_gpu": T, "bins": G, "pairs": P, "n_fft": sc.n_fft,
                   "topk": sc.topk,
                   "l2": "flushed between timed steps (512 MB write, outside the events)",
                   "parallelism": f"trial-sharded x{world}"},
        "trials_per_s": T * world / (ms * 1e-3),
        "wall_ms_per_step": t_wall * 1e3 / args.steps,
        "kernel_timing": "per-kernel CUDA events on the launching stream, in a second pass of "
                         "the same steps (the headline pass has only the step events)",
        "kernels_ms": kernels_ms,
        "launches_per_step": {k: v[1] / args.steps for k, v in kern.items() if v[1]},
        "roofline": {"bound": "smem", "achieved": achieved, "peak": smem_peak, "unit": "GB/s",
                     "frac": achieved / smem_peak,
                     "traffic": ncu_traffic(sc.name, t_launch),
                     "launch_ms": g_launch_ms, "trials_per_launch": t_launch,
                     "traffic_note": "DRAM read+write bytes per launch from the committed ncu "
                                     "--set full capture (profiles/), compare with hbm."
                                     "bytes_per_launch",
                     "kernel": GATHER_LABEL.get(sc.name, "k_gather"),
                     "peak_source": "measured in-run (gh_measure_smem_peak, LDS.128 all SMs)",
                     "algorithmic_bytes_per_launch": lsu_bytes,
                     "unit_bytes": "4 B of shared-memory power per bin x pair x trial (K = 1), "
                                   "24 B (3 complex64) for K = 3",
                     "hbm": {"bytes_per_launch": hbm_bytes,
                             "achieved_gbs": hbm_bytes / (g_launch_ms * 1e-3) / 1e9,
                             "peak_gbs": pk.get("hbm_gbs")}},
        "e2e": {"value": units_step / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": T * P * N * 16, "d2h_bytes_per_step": T * kk * (8 + 4),
                "ms_per_step": e2e_s * 1e3,
                "api": ("gh_hop_estimate_topk" if topk else "gh_hop_estimate")
                       + " (host complex128 frames, pinned)",
                "h2d_gbs_raw": h2d_gbs,
                "h2d_bound_ms": T * P * N * 16 / (h2d_gbs * 1e9) * 1e3},
        "campaign": {"ms_per_step": camp_ms, "trials_per_s": T * world / (camp_ms * 1e-3),
                     "value": units_step / (camp_ms * 1e-3),
                     "api": ("gh_campaign_hop_topk_d" if topk else "gh_campaign_hop_d")
                            + " (synthesis fused into the FFT)"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if direct:
        line["direct"] = direct
    if indirect:
        line["indirect"] = indirect
    if not args.no_stats:
        line["statistics"] = campaign_statistics(ctx, sc, T)
    if world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        oi, oc, _ = O.build_table(sc)
        line["cpu_baseline"] = cpu_baseline(sc, oi, oc)
    print(json.dumps(line), flush=True)
    if dist:
        tdist.destroy_process_group()


def campaign_statistics(ctx, sc, T):
    """Error statistics of the config through the device campaign driver
    (gh_campaign_run = run_monte_carlo, montecarlo.cpp:99-179), outside the
    timed regions: BASELINE c2 "run both ways" (hop and direct: RMSE, fraction
    within 1 m), the c4 SNR sweep (-10..20 dB), c3's K-target assignment
    statistics. The parity tests compare the same numbers with the oracle
    campaign (tests/test_gpu_parity_full.py, tests/test_campaign.py)."""
    import paper_2307_16550_b200 as gh
    kw = {}
    if sc.name in ("c1", "c2"):
        kw["algorithms"] = ("hop", "direct")
    if sc.name == "c4":
        kw["snr_db"] = [-10.0, -5.0, 0.0, 5.0, 10.0, 15.0, 20.0]
    cells = gh.campaign_run(ctx, sc, n_trials=T, thresholds=[1.0], **kw)
    out = []
    for c in cells:
        n = max(c["estimates"], 1)
        out.append({"algorithm": c["algorithm"],
                    "snr_db": None if c["snr_db"] != c["snr_db"] else c["snr_db"],
                    "trials": c["trials"], "rmse_m": c["rmse_m"],
                    "within_1m": c["hit_ratio"][0], "within_half_resolution": c["hits_half_res"] / n,
                    "online_ms": c["online_ms"]})
    return {"api": "gh_campaign_run (device campaign driver, statistics on the device)",
            "topk": sc.topk, "cells": out}


def run_grid_sharded(args, world, rank, local):
    """BASELINE c5: the location grid is sharded across ranks (z layers);
    every rank synthesises the same trials (no signal traffic) and scans its
    slab. K = 3 targets: each rank's halo shard reports the top-3 local maxima
    of its core layers (one extra layer each side completes the border
    neighbourhoods), one NCCL all-gather of the K int64 keys per trial
    (value bits << 32 | 2^32-1-bin) and a top-K over them merge the shards
    exactly. value = full-grid units / step."""
    import torch
    import paper_2307_16550_b200 as gh
    from paper_2307_16550_b200 import distributed as D
    from paper_2307_16550_b200 import scene as S

    dist = world > 1
    if dist:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    sc = S.baseline(args.config)
    K = sc.topk
    T = args.trials or 256
    lo, hi = D.shard(sc.slab_axis_len(), world, rank)
    ctx = gh.Context(local)
    t_build = time.perf_counter()
    table = gh.precompute_hop_table_shard(ctx, sc, lo, hi, halo=dist)
    ctx.synchronize()
    t_build = time.perf_counter() - t_build
    dev = f"cuda:{local}"
    stream = ctx.torch_stream()
    gathered = torch.empty((world, T, K), dtype=torch.int64, device=dev)

    def step(k):
        idx, val = gh.campaign_hop_topk(ctx, table, sc, k * T, T, K)
        # key = float bits << 32 | (2^32 - 1 - bin), -1 = no maximum
        keys = torch.where(idx >= 0, (val.view(torch.int32).to(torch.int64) << 32) | (0xFFFFFFFF - idx),
                           torch.full_like(idx, -1))
        if dist:
            tdist.all_gather_into_tensor(gathered, keys)
            keys = torch.topk(gathered.permute(1, 0, 2).reshape(T, world * K), K, dim=1).values
        return keys

    with torch.cuda.stream(stream):
        for k in range(max(3, args.warmup)):
            step(k)
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            e0.record(stream)
            for k in range(args.steps):
                keys = step(k)
            e1.record(stream)
        torch.cuda.synchronize()
    launches = ctx.launches - launches0
    ms = D.max_over_ranks(e0.elapsed_time(e1) / args.steps, device=dev)
    if dist:
        tdist.barrier()
    # per-kernel CUDA events in a second pass of the same steps
    smem_peak = ctx.smem_peak_gbps()
    ctx.reset_timing()
    ctx.set_timing(not args.no_kernel_timing)
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            step(k)
    ctx.synchronize()
    ctx.set_timing(False)
    kern = {name: ctx.kernel_time(name) for name in ("synth_fft", "gather", "topk")}
    g_ms, g_n = kern["gather"]
    if rank == 0:
        units = T * sc.units_per_trial()
        shard_units = units * (table.n_bins / sc.n_bins)  # this rank's slab (+ halo layers)
        g_launch = max(g_ms / max(g_n, 1), 1e-9)
        lsu_bytes = shard_units / max(1, g_n // args.steps) * 4.0
        line = {
            "metric": METRIC, "value": units / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
            "data": f"synthetic (counter-based RNG, seed 20260816), {sc.name} scene",
            "config": {"workload": f"{sc.name}: {T} trials/step, {sc.n_bins} bins x {sc.n_pairs} "
                                   f"pairs, N={sc.n_samples}, M={sc.n_fft}, top-{K} local maxima, "
                                   f"location grid sharded over {world} GPU(s) "
                                   f"({sc.slab_axis_len()} z layers, 1-layer halos)",
                       "trials_per_step": T, "bins": sc.n_bins, "pairs": sc.n_pairs, "topk": K,
                       "parallelism": f"grid-sharded x{world}"},
            "trials_per_s": T / (ms * 1e-3),
            "table_build_s_rank0": t_build,
            "kernels_ms": {k: v[0] / args.steps for k, v in kern.items() if v[1]},
            "roofline": {"bound": "smem", "achieved": lsu_bytes / (g_launch * 1e-3) / 1e9,
                         "peak": smem_peak, "unit": "GB/s",
                         "frac": lsu_bytes / (g_launch * 1e-3) / 1e9 / smem_peak,
                         "kernel": "k_gather_tiled (64 pairs, map mode) + k_topk_localmax (3-D)",
                         "launch_ms": g_launch, "traffic": None,
                         "peak_source": "measured in-run (gh_measure_smem_peak, LDS.128 all SMs)",
                         "algorithmic_bytes_per_launch": lsu_bytes},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        tdist.destroy_process_group()


def relaunch(args) -> int:
    """`--gpus N` outside torch.distributed.run: start one rank per GPU
    (127.0.0.1 rendezvous) and return their exit status."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--trials", type=int, default=0)
    ap.add_argument("--ref-trials", type=int, default=0,
                    help="reference arm: cap on trials per step (default: time-bounded)")
    ap.add_argument("--ref-seconds", type=float, default=90.0,
                    help="reference arm: CPU seconds for warmup + steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-direct", action="store_true")
    ap.add_argument("--no-stats", action="store_true",
                    help="skip the campaign statistics section (RMSE / hit ratios)")
    ap.add_argument("--direct-steps", type=int, default=3)
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="diagnostic: no per-kernel CUDA events inside the timed steps")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    elif args.config == "c5":
        run_grid_sharded(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
