"""Independent numpy fp64 restatement of the reference hot path.

TEST INFRASTRUCTURE ONLY — a second, differently written oracle used to
cross-check oracle/gridhop_oracle.cpp (vectorised numpy instead of scalar
loops; numpy.fft (pocketfft) instead of the C radix-2 FFT).

Anchors (reference, /root/reference/proj/core): fit_atom interp.cpp:78-154,
atom_kernel interp.cpp:21-37 (evaluated here in closed form), hop_bin_value
hopping.cpp:59-102, location_decision_map direct.cpp:90-144, sample_scene
montecarlo.cpp:48-66, synthesize_frame/add_noise synth.cpp:15-49.
"""
from __future__ import annotations

import math

import numpy as np

from paper_2307_16550_b200.scene import substream, uniform, Scene

TWO_PI = 2.0 * math.pi


def atom_kernel(delta, n: int):
    """D(delta) = sum_{m<n} exp(j 2pi delta m / n), closed form (geometric sum)."""
    m = np.arange(n)
    return np.exp(1j * TWO_PI * np.multiply.outer(np.asarray(delta, dtype=np.float64), m) / n).sum(-1)


def wrap_range(r: float, n: int) -> float:
    w = math.fmod(r, n)
    if w < 0:
        w += n
    if w >= n:
        w = 0.0
    return w


def fit_atom(n: int, os_: int, r: float, scheme: int):
    """(indices, coefficients, residual) — same rules as interp.cpp:78-154 +
    the polar scheme, solved with numpy.linalg.solve instead of LLT."""
    M = n * os_
    rw = wrap_range(r, n)
    pos = rw * os_
    if scheme == 1:
        idx = np.array([int(round_half_away(pos)) % M])
        c = np.array([1.0 + 0j])
    elif scheme == 2:
        i0 = math.floor(pos)
        t = pos - i0
        idx = np.array([i0 % M, (i0 + 1) % M])
        c = np.array([1 - t, t], dtype=complex)
    else:
        i = int(round_half_away(pos))
        idx = np.array([(i - 1) % M, i % M, (i + 1) % M])
        c = None
    rbar = idx / os_
    G = atom_kernel(rbar[:, None] - rbar[None, :], n)
    b = atom_kernel(rbar - rw, n)
    if scheme == 3:
        c = np.linalg.solve(G, b)
    elif scheme == 4:
        h = 1.0 / os_
        d1 = math.sqrt(max(0.0, 2 * n - 2 * atom_kernel(h, n).real))
        d2 = math.sqrt(max(0.0, 2 * n - 2 * atom_kernel(2 * h, n).real))
        theta = 2 * math.acos(min(1.0, max(-1.0, d2 / (2 * d1))))
        t = pos - round_half_away(pos)
        a = (1 - math.cos(theta * t)) / (1 - math.cos(theta))
        bb = math.sin(theta * t) / (2 * math.sin(theta))
        c = np.array([0.5 * a - bb, 1 - a, 0.5 * a + bb], dtype=complex)
    quad = np.vdot(c, G @ c).real
    cross = np.vdot(c, b).real
    res = math.sqrt(max(0.0, n - 2 * cross + quad))
    return idx, c, res


def round_half_away(x: float) -> float:
    """llround semantics (half away from zero)."""
    return math.floor(x + 0.5) if x >= 0 else -math.floor(-x + 0.5)


def sensed_ranges(scene: Scene, x: np.ndarray) -> np.ndarray:
    """[..., P] ranges in fast-time bins for points x [..., 3]."""
    d_tx = np.linalg.norm(x[..., None, :] - scene.tx, axis=-1)
    d_rx = np.linalg.norm(x[..., None, :] - scene.rx, axis=-1)
    return scene.range_scale * (d_tx + d_rx)


def scene_draws(scene: Scene, trial: int):
    K, P, D = scene.n_targets, scene.n_pairs, scene.dims
    key = substream(scene.seed, trial, 0x53434E)
    tg = np.zeros((K, 3))
    for k in range(K):
        for d in range(3):
            tg[k, d] = scene.area_lo[d]
            if d < D:
                tg[k, d] = scene.area_lo[d] + (scene.area_hi[d] - scene.area_lo[d]) * uniform(key, k * D + d)
    al = np.zeros((K, P), dtype=complex)
    for k in range(K):
        for p in range(P):
            pp = 0 if scene.amp_mode in (0, 2) else p
            at = K * D + 2 * (k * P + pp)
            u0, u1 = uniform(key, at), uniform(key, at + 1)
            if scene.amp_mode in (0, 1):
                al[k, p] = np.exp(1j * TWO_PI * u0)
            else:
                al[k, p] = math.sqrt(-math.log1p(-u0)) * np.exp(1j * TWO_PI * u1)
    sig = np.zeros(P)
    for p in range(P):
        if scene.snr_mode == 0:
            sig[p] = 10 ** (-scene.snr_db / 20)
        elif scene.snr_mode == 1:
            u = uniform(key, K * D + 2 * K * P + p)
            sig[p] = 10 ** (-(scene.snr_lo + (scene.snr_hi - scene.snr_lo) * u) / 20)
    return tg, al, sig


def synth(scene: Scene, trial: int) -> np.ndarray:
    tg, al, sig = scene_draws(scene, trial)
    N, P = scene.n_samples, scene.n_pairs
    n = np.arange(N)
    r = sensed_ranges(scene, tg)  # [K, P]
    y = (al[:, :, None] * np.exp(1j * TWO_PI * r[:, :, None] * n / N)).sum(0)
    for p in range(P):
        if sig[p] == 0:
            continue
        key = substream(scene.seed, trial, p)
        u1 = np.array([uniform(key, 2 * i) for i in range(N)])
        u2 = np.array([uniform(key, 2 * i + 1) for i in range(N)])
        y[p] += sig[p] * np.sqrt(-np.log1p(-u1)) * np.exp(1j * TWO_PI * u2)
    return y


def spectra(frames: np.ndarray, m: int) -> np.ndarray:
    return np.fft.fft(frames, n=m, axis=-1)


def hop_map(spec: np.ndarray, idx: np.ndarray, coef: np.ndarray, magnitude=False) -> np.ndarray:
    """spec [T, P, M]; idx/coef [G, P, K] -> [T, G]."""
    P = spec.shape[1]
    z = spec[:, np.arange(P)[None, :, None], idx]  # [T, G, P, K]
    v = (coef[None] * z).sum(-1)
    pw = np.abs(v) ** 2
    return (np.sqrt(pw) if magnitude else pw).sum(-1)


def direct_map(scene: Scene, frames: np.ndarray, magnitude=False) -> np.ndarray:
    x = scene.grid_points(np.arange(scene.n_bins))
    r = sensed_ranges(scene, x)  # [G, P]
    N = scene.n_samples
    n = np.arange(N)
    out = np.zeros((frames.shape[0], scene.n_bins))
    for p in range(scene.n_pairs):
        A = np.exp(-1j * TWO_PI * np.outer(r[:, p], n) / N)  # conj atoms [G, N]
        z = frames[:, p, :] @ A.T
        pw = np.abs(z) ** 2
        out += np.sqrt(pw) if magnitude else pw
    return out
