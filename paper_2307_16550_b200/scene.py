"""Scene / campaign descriptions and the five BASELINE configurations.

Mirrors the reference's WaveformConfig + SceneGeometry + LocationGrid +
Scenario (include/gridhop/model.hpp:21-111, scenario.hpp), generalised to a
list of (TX, RX) pairs in 3-D (BASELINE c3-c5 use several TX, c5 is 3-D).

Units follow the reference: ranges are in fast-time bins of the N-point DFT,
r = (B / c) * (|x - tx| + |x - rx|) (src/model.cpp:45-52); one bin of the
M = os * N zero-padded FFT is c * N / (B * M) metres of summed path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace

import numpy as np

SPEED_OF_LIGHT = 299792458.0  # model.hpp:18

NEAREST, LINEAR, POLY3, POLAR = 1, 2, 3, 4
SCHEME_NAMES = {NEAREST: "nearest", LINEAR: "linear", POLY3: "poly3", POLAR: "polar"}
SCHEME_ORDER = {NEAREST: 1, LINEAR: 2, POLY3: 3, POLAR: 3}
POWER, MAGNITUDE = 0, 1

# amplitude / SNR models of the campaign (gh_campaign)
AMP_UNIT_SHARED, AMP_UNIT_PER_PAIR, AMP_CGAUSS_SHARED, AMP_CGAUSS_PER_PAIR = 0, 1, 2, 3
SNR_FIXED, SNR_UNIFORM_PER_PAIR, SNR_NOISELESS = 0, 1, 2

BASE_SEED = 20260816  # proj/scenarios/comparison.scn:24
GEOMETRY_TAG = 0x47454F  # substream tag for random station placement


def scheme_from_name(name: str) -> int:
    """scheme_from_name (src/interp.cpp:58-65) + polar."""
    for k, v in SCHEME_NAMES.items():
        if v == name:
            return k
    raise ValueError(f"unknown interpolation scheme '{name}' (valid: nearest, linear, poly3, polar)")


# ---------------------------------------------------------------- ctypes structs
class CWave(C.Structure):
    _fields_ = [("n_samples", C.c_int32), ("os_range", C.c_int32), ("range_scale", C.c_double),
                ("n_pairs", C.c_int32), ("tx", C.POINTER(C.c_double)), ("rx", C.POINTER(C.c_double))]


class CGrid(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("spacing", C.c_double * 3), ("n", C.c_int32 * 3)]


class CCampaign(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_targets", C.c_int32), ("dims", C.c_int32),
                ("area_lo", C.c_double * 3), ("area_hi", C.c_double * 3),
                ("amp_mode", C.c_int32), ("snr_mode", C.c_int32), ("snr_db", C.c_double),
                ("snr_lo", C.c_double), ("snr_hi", C.c_double)]


# ---------------------------------------------------------------- rng (host copy)
_M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """rng.hpp:11-16."""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def substream(seed: int, a: int, b: int) -> int:
    """rng.hpp:20-25."""
    x = splitmix64(seed ^ 0x6A09E667F3BCC909)
    x = splitmix64((x + 0x9E3779B97F4A7C15 * (a + 1)) & _M64)
    x = splitmix64((x + 0xBF58476D1CE4E5B9 * (b + 1)) & _M64)
    return x


def uniform(key: int, counter: int) -> float:
    """Draw `counter` of the SplitMix64 stream seeded with `key`, [0, 1)."""
    v = splitmix64((key + 0x9E3779B97F4A7C15 * counter) & _M64)
    return (v >> 11) * 2.0 ** -53


@dataclass
class Scene:
    name: str
    n_samples: int
    os_range: int
    bandwidth: float
    tx: np.ndarray            # [P, 3]
    rx: np.ndarray            # [P, 3]
    grid_origin: tuple
    grid_spacing: tuple
    grid_n: tuple
    trials: int = 1000
    seed: int = BASE_SEED
    n_targets: int = 1
    dims: int = 2
    area_lo: tuple = (0.0, 0.0, 0.0)
    area_hi: tuple = (0.0, 0.0, 0.0)
    amp_mode: int = AMP_UNIT_PER_PAIR
    snr_mode: int = SNR_FIXED
    snr_db: float = 10.0
    snr_lo: float = 0.0
    snr_hi: float = 0.0
    scheme: int = NEAREST
    wrap: bool = True
    combine: int = POWER
    topk: int = 1
    snr_sweep: tuple = ()
    c: float = SPEED_OF_LIGHT
    notes: str = ""
    _keep: list = field(default_factory=list, repr=False)

    # ---- derived sizes
    @property
    def n_pairs(self) -> int:
        return int(self.tx.shape[0])

    @property
    def n_fft(self) -> int:
        return self.n_samples * self.os_range

    @property
    def n_bins(self) -> int:
        return int(self.grid_n[0]) * int(self.grid_n[1]) * int(self.grid_n[2])

    @property
    def range_scale(self) -> float:
        """WaveformConfig::range_scale (model.hpp:36): bins per metre."""
        return self.bandwidth / self.c

    @property
    def k(self) -> int:
        return SCHEME_ORDER[self.scheme]

    def with_(self, **kw) -> "Scene":
        return replace(self, **kw)

    # ---- C views (arrays kept alive on the instance)
    def c_wave(self) -> CWave:
        tx = np.ascontiguousarray(self.tx, dtype=np.float64)
        rx = np.ascontiguousarray(self.rx, dtype=np.float64)
        self._keep[:] = [tx, rx]
        return CWave(self.n_samples, self.os_range, self.range_scale, self.n_pairs,
                     tx.ctypes.data_as(C.POINTER(C.c_double)),
                     rx.ctypes.data_as(C.POINTER(C.c_double)))

    def c_grid(self) -> CGrid:
        g = CGrid()
        for d in range(3):
            g.origin[d] = float(self.grid_origin[d])
            g.spacing[d] = float(self.grid_spacing[d])
            g.n[d] = int(self.grid_n[d])
        return g

    def c_campaign(self, snr_db: float | None = None) -> CCampaign:
        c = CCampaign()
        c.seed = self.seed
        c.n_targets = self.n_targets
        c.dims = self.dims
        for d in range(3):
            c.area_lo[d] = float(self.area_lo[d])
            c.area_hi[d] = float(self.area_hi[d])
        c.amp_mode = self.amp_mode
        c.snr_mode = self.snr_mode
        c.snr_db = float(self.snr_db if snr_db is None else snr_db)
        c.snr_lo = float(self.snr_lo)
        c.snr_hi = float(self.snr_hi)
        return c

    # ---- geometry helpers (host, fp64; identical rounding to the oracle)
    def grid_point(self, k: int) -> np.ndarray:
        nx, ny = int(self.grid_n[0]), int(self.grid_n[1])
        ix, iy, iz = k % nx, (k // nx) % ny, k // (nx * ny)
        return np.array([self.grid_origin[0] + self.grid_spacing[0] * ix,
                         self.grid_origin[1] + self.grid_spacing[1] * iy,
                         self.grid_origin[2] + self.grid_spacing[2] * iz])

    def grid_points(self, idx) -> np.ndarray:
        idx = np.asarray(idx, dtype=np.int64)
        nx, ny = int(self.grid_n[0]), int(self.grid_n[1])
        ix, iy, iz = idx % nx, (idx // nx) % ny, idx // (nx * ny)
        o, s = self.grid_origin, self.grid_spacing
        return np.stack([o[0] + s[0] * ix, o[1] + s[1] * iy, o[2] + s[2] * iz], axis=-1)

    def alias_fraction(self, sample: int = 200_000) -> float:
        """Fraction of (bin, pair) entries whose sensed range leaves [0, N)."""
        G = self.n_bins
        rng = np.random.default_rng(0)
        ks = np.arange(G) if G <= sample else rng.integers(0, G, sample)
        x = self.grid_points(ks)
        r = self.range_scale * (np.linalg.norm(x[:, None, :] - self.tx[None], axis=-1)
                                + np.linalg.norm(x[:, None, :] - self.rx[None], axis=-1))
        return float(np.mean((r < 0) | (r >= self.n_samples)))

    def units_per_trial(self) -> int:
        """Gather units (bin x pair correlations) per trial, SURVEY §8(d)."""
        return self.n_bins * self.n_pairs

    def slab_axis_len(self) -> int:
        """Length of the axis location-grid shards split: z (3-D) or y (2-D)."""
        return int(self.grid_n[2]) if int(self.grid_n[2]) > 1 else int(self.grid_n[1])

    def slab_bins(self, lo: int, hi: int) -> tuple[int, int]:
        """Global bin range [b0, b1) of layers [lo, hi) (contiguous, x fastest)."""
        layer = int(self.grid_n[0]) * (int(self.grid_n[1]) if int(self.grid_n[2]) > 1 else 1)
        return lo * layer, hi * layer


def _circle(radius: float, angles_deg) -> np.ndarray:
    a = np.deg2rad(np.asarray(angles_deg, dtype=np.float64))
    return np.stack([radius * np.cos(a), radius * np.sin(a), np.zeros_like(a)], axis=-1)


def _random_circle(n: int, radius: float, tag_b: int, seed: int = BASE_SEED) -> np.ndarray:
    key = substream(seed, 0, GEOMETRY_TAG + tag_b)
    ang = np.array([2.0 * math.pi * uniform(key, i) for i in range(n)])
    return np.stack([radius * np.cos(ang), radius * np.sin(ang), np.zeros(n)], axis=-1)


def _random_square_perimeter(n: int, half: float, zmax: float, tag_b: int,
                             seed: int = BASE_SEED) -> np.ndarray:
    key = substream(seed, 0, GEOMETRY_TAG + tag_b)
    out = []
    for i in range(n):
        s = 8.0 * half * uniform(key, 2 * i)  # arc length along the perimeter
        z = zmax * uniform(key, 2 * i + 1)
        side, off = int(s // (2 * half)), s % (2 * half) - half
        x, y = [(off, -half), (half, off), (-off, half), (-half, -off)][min(side, 3)]
        out.append((x, y, z))
    return np.array(out, dtype=np.float64)


def _pairs(tx: np.ndarray, rx: np.ndarray):
    """All TX x RX pairs, TX-major."""
    P = tx.shape[0] * rx.shape[0]
    return np.repeat(tx, rx.shape[0], axis=0).reshape(P, 3), np.tile(rx, (tx.shape[0], 1))


def baseline(name: str) -> Scene:
    """The five BASELINE.json configs (SURVEY.md §8(d) makes them concrete)."""
    if name in ("c1", "c2"):
        tx = np.zeros((3, 3))
        rx = _circle(50.0, [0.0, 120.0, 240.0])
        return Scene(name=name, n_samples=256, os_range=4, bandwidth=1e9, tx=tx, rx=rx,
                     grid_origin=(-49.75, -49.75, 0.0), grid_spacing=(0.5, 0.5, 1.0),
                     grid_n=(200, 200, 1), trials=1000 if name == "c1" else 10000,
                     n_targets=1, dims=2, area_lo=(-50.0, -50.0, 0.0), area_hi=(50.0, 50.0, 0.0),
                     amp_mode=AMP_UNIT_PER_PAIR, snr_mode=SNR_FIXED, snr_db=10.0,
                     scheme=NEAREST, wrap=True, combine=POWER,
                     notes="1 TX + 3 RX, 67.7% of entries alias -> wrap mode")
    if name == "c3":
        tx, rx = _pairs(_random_circle(2, 60.0, 1), _random_circle(8, 60.0, 2))
        return Scene(name=name, n_samples=1024, os_range=4, bandwidth=1e9, tx=tx, rx=rx,
                     grid_origin=(-49.95, -49.95, 0.0), grid_spacing=(0.1, 0.1, 1.0),
                     grid_n=(1000, 1000, 1), trials=100000, n_targets=5, dims=2,
                     area_lo=(-50.0, -50.0, 0.0), area_hi=(50.0, 50.0, 0.0),
                     amp_mode=AMP_CGAUSS_PER_PAIR, snr_mode=SNR_UNIFORM_PER_PAIR,
                     snr_lo=0.0, snr_hi=20.0, scheme=NEAREST, wrap=False, topk=5,
                     notes="2 TX x 8 RX on a 60 m circle, bandwidth assumed 1 GHz")
    if name == "c4":
        tx, rx = _pairs(_random_circle(4, 40.0, 3), _random_circle(4, 40.0, 4))
        return Scene(name=name, n_samples=512, os_range=2, bandwidth=1e9, tx=tx, rx=rx,
                     grid_origin=(-49.9, -49.9, 0.0), grid_spacing=(0.2, 0.2, 1.0),
                     grid_n=(500, 500, 1), trials=20000, n_targets=1, dims=2,
                     area_lo=(-50.0, -50.0, 0.0), area_hi=(50.0, 50.0, 0.0),
                     amp_mode=AMP_UNIT_PER_PAIR, snr_mode=SNR_FIXED, snr_db=10.0,
                     scheme=POLAR, wrap=True, snr_sweep=(-10.0, -5.0, 0.0, 5.0, 10.0, 15.0, 20.0),
                     notes="4 TX x 4 RX on a 40 m circle, bandwidth assumed 1 GHz")
    if name == "c5":
        tx, rx = _pairs(_random_square_perimeter(8, 50.0, 10.0, 5),
                        _random_square_perimeter(8, 50.0, 10.0, 6))
        sx, sz = 100.0 / 512, 20.0 / 64
        return Scene(name=name, n_samples=512, os_range=4, bandwidth=1e9, tx=tx, rx=rx,
                     grid_origin=(-50.0 + sx / 2, -50.0 + sx / 2, sz / 2),
                     grid_spacing=(sx, sx, sz), grid_n=(512, 512, 64), trials=10000,
                     n_targets=3, dims=3, area_lo=(-50.0, -50.0, 0.0),
                     area_hi=(50.0, 50.0, 20.0), amp_mode=AMP_UNIT_PER_PAIR,
                     snr_mode=SNR_FIXED, snr_db=10.0, scheme=NEAREST, wrap=True, topk=3,
                     notes="8 TX x 8 RX on the 100 m square perimeter, heights 0-10 m")
    raise ValueError(f"unknown config {name!r}")


def small(name: str = "small", P: int = 3, N: int = 64, os: int = 4, nx: int = 24, ny: int = 20,
          scheme: int = NEAREST, wrap: bool = True, seed: int = 7, **kw) -> Scene:
    """A small c1-like scene that the fp64 oracle finishes in milliseconds."""
    rx = _circle(30.0, np.linspace(0.0, 360.0, P, endpoint=False) + 10.0)
    tx = np.tile(np.array([[1.0, -2.0, 0.0]]), (P, 1))
    sp = 0.6
    ox, oy = -sp * (nx - 1) / 2, -sp * (ny - 1) / 2
    base = dict(name=name, n_samples=N, os_range=os, bandwidth=250e6, tx=tx, rx=rx,
                grid_origin=(ox, oy, 0.0), grid_spacing=(sp, sp, 1.0), grid_n=(nx, ny, 1),
                trials=37, seed=seed, n_targets=1, dims=2,
                area_lo=(ox - sp / 2, oy - sp / 2, 0.0), area_hi=(-ox + sp / 2, -oy + sp / 2, 0.0),
                amp_mode=AMP_UNIT_PER_PAIR, snr_mode=SNR_FIXED, snr_db=10.0, scheme=scheme,
                wrap=wrap)
    base.update(kw)
    return Scene(**base)
