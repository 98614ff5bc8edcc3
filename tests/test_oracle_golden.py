"""CPU: pin the fp64 oracle (oracle/) before trusting it.

1. Known answers asserted by the reference's own tests
   (tests/golden/reference_known_answers.json, each entry cites its source).
2. Property tests the reference runs (Cauchy-Schwarz hop-vs-direct bound,
   map == pointwise reads, thread invariance, window errors).
3. Cross-check against an independent numpy restatement (oracle/oracle_np.py).
4. Regression against the committed golden fixture (tests/golden/*.npz made
   by tests/golden/make_golden.py).
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from oracle import oracle_np as ONP
from paper_2307_16550_b200 import scene as S

GOLD = Path(__file__).resolve().parent / "golden"
KA = json.loads((GOLD / "reference_known_answers.json").read_text())
SCHEMES = {"nearest": S.NEAREST, "linear": S.LINEAR, "poly3": S.POLY3, "polar": S.POLAR}


def test_fit_atom_known_answers():
    for case in KA["fit_atom"]:
        idx, c, res = O.fit_atom(case["n"], case["os"], case["r"], SCHEMES[case["scheme"]])
        if "indices" in case:
            assert list(idx) == case["indices"], case["cite"]
        if "coeffs" in case:
            want = np.array([complex(*z) for z in case["coeffs"]])
            assert np.abs(c - want).max() <= case.get("tol", 0.0), case["cite"]
        if "same_as_r" in case:
            i2, c2, _ = O.fit_atom(case["n"], case["os"], case["same_as_r"], SCHEMES[case["scheme"]])
            assert np.array_equal(idx, i2) and np.abs(c - c2).max() < 1e-12


def naive_residual(idx, c, n, os_, r):
    m = np.arange(n)
    a = np.exp(2j * np.pi * r * m / n)
    for j in range(len(idx)):
        a = a - np.conj(c[j]) * np.exp(2j * np.pi * (idx[j] / os_) * m / n)
    return np.linalg.norm(a)


def test_residual_closed_form_and_order():
    ka = KA["residual_order"]
    res = {}
    for name in ("nearest", "linear", "poly3", "polar"):
        idx, c, r = O.fit_atom(ka["n"], ka["os"], ka["r"], SCHEMES[name])
        assert r == pytest.approx(naive_residual(idx, c, ka["n"], ka["os"], ka["r"]), rel=1e-6)
        res[name] = r
    assert res["poly3"] < res["linear"] < res["nearest"]
    # polar sits between least squares and linear
    assert res["poly3"] <= res["polar"] < res["nearest"]


def test_ongrid_fits_are_unit_vectors():
    ka = KA["ongrid_unit_vectors"]
    for name in ("nearest", "linear", "poly3", "polar"):
        for b in ka["bins"]:
            idx, c, res = O.fit_atom(ka["n"], ka["os"], b / ka["os"], SCHEMES[name])
            want = np.where(idx == b, 1.0, 0.0)
            assert np.abs(c - want).max() < ka["tol"], (name, b)
            assert res < ka["residual_tol"]


def test_combined_coefficients_bound():
    # test_interp.cpp:132-158: |sum c_j Z[I_j] - <y, a(r)>| <= residual ||y||
    rng = np.random.default_rng(61)
    y = rng.uniform(-1, 1, 64) + 1j * rng.uniform(-1, 1, 64)
    z = O.spectra(y[None], 256)[0]
    m = np.arange(64)
    for r in (5.37, 20.11, 63.93):
        for scheme in (S.POLY3, S.POLAR, S.LINEAR, S.NEAREST):
            idx, c, res = O.fit_atom(64, 4, r, scheme)
            want = np.sum(y * np.exp(-2j * np.pi * r * m / 64))
            assert abs(np.sum(c * z[idx]) - want) <= res * np.linalg.norm(y) + 1e-9


def test_argmax_known_answers():
    for case in KA["argmax"]:
        assert O.argmax(np.array(case["values"], dtype=float)) == case["index"]
    with pytest.raises(O.OracleError):
        O.argmax(np.array([]))


def test_sensed_range_known_answers():
    ka = KA["sensed_range"]
    scale = ka["bandwidth"] / S.SPEED_OF_LIGHT
    for case in ka["cases"]:
        r = O.sensed_range(scale, ka["tx"] + [0.0], case["rx"] + [0.0], case["x"] + [0.0])
        assert r == pytest.approx(scale * case["summed_path_m"], rel=ka["rel_tol"])
    with pytest.raises(O.OracleError, match="degenerate geometry"):
        O.sensed_range(scale, [0, 0, 0], [1, 0, 0], [0, 0, 0])


def test_range_resolution():
    ka = KA["range_resolution"]
    assert S.SPEED_OF_LIGHT / (2 * ka["bandwidth"]) == pytest.approx(ka["metres"], abs=ka["tol"])


def test_noise_sigma_and_power():
    for case in KA["noise_sigma"]:
        assert case["alpha_ref"] * 10 ** (-case["snr_db"] / 20) == pytest.approx(case["sigma"])
    sc = S.small(N=256, snr_mode=S.SNR_FIXED, snr_db=0.0, seed=7)
    fr, _ = O.synth(sc, 0, 8)
    clean, _ = O.synth(sc.with_(snr_mode=S.SNR_NOISELESS), 0, 8)
    pw = np.mean(np.abs(fr - clean) ** 2)
    assert pw == pytest.approx(1.0, rel=KA["noise_power"]["rel_tol"])


def test_noise_paired_across_snr_and_deterministic():
    ka = KA["noise_paired_across_snr"]
    a, _ = O.synth(S.small(snr_db=ka["snr_a"]), 3, 2)
    b, _ = O.synth(S.small(snr_db=ka["snr_b"]), 3, 2)
    clean, _ = O.synth(S.small(snr_mode=S.SNR_NOISELESS), 3, 2)
    ratio = 10 ** ((ka["snr_b"] - ka["snr_a"]) / 20)
    assert np.abs((a - clean) - ratio * (b - clean)).max() < ka["tol"]
    a2, _ = O.synth(S.small(snr_db=ka["snr_a"]), 3, 2)
    assert np.array_equal(a, a2)
    c, _ = O.synth(S.small(snr_db=ka["snr_a"]), 4, 2)
    assert np.abs(a[0] - c[0]).max() > 1e-6


def test_fft_vs_literal_dft():
    rng = np.random.default_rng(3)
    for n, m in ((64, 256), (16, 16), (24, 40)):  # includes a non power of two
        y = rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n))
        z = O.spectra(y, m)
        k = np.arange(m)[:, None]
        s = np.arange(n)[None, :]
        lit = y @ np.exp(-2j * np.pi * k * s / m).T
        assert np.abs(z - lit).max() < KA["fft_vs_dft_abs_tol"]["tol"] * 10
        assert np.abs(z - np.fft.fft(y, n=m)).max() < 1e-10


def test_fft_range_grid():
    ka = KA["fft_range_grid"]
    grid = np.arange(ka["n"] * ka["os"]) / ka["os"]
    assert grid.size == ka["size"]
    for k, v in ka["values"].items():
        assert grid[int(k)] == v


@pytest.mark.parametrize("scheme", [S.NEAREST, S.LINEAR, S.POLY3, S.POLAR])
def test_oracle_matches_numpy_restatement(scheme):
    sc = S.small(scheme=scheme, nx=9, ny=7)
    idx, coef, _ = O.build_table(sc)
    for b in range(0, sc.n_bins, 5):
        x = sc.grid_point(b)
        for p in range(sc.n_pairs):
            r = O.sensed_range(sc.range_scale, sc.tx[p], sc.rx[p], x)
            i2, c2, _ = ONP.fit_atom(sc.n_samples, sc.os_range, r, scheme)
            assert np.array_equal(idx[b, p], i2)
            assert np.abs(coef[b, p] - c2).max() < 1e-9
    fr, _ = O.synth(sc, 0, 3)
    for t in range(3):
        assert np.abs(fr[t] - ONP.synth(sc, t)).max() < 1e-9
    sp = O.spectra(fr, sc.n_fft)
    assert np.abs(sp - ONP.spectra(fr, sc.n_fft)).max() < 1e-9
    m1 = O.hop_map(sp, idx, coef)
    assert np.abs(m1 - ONP.hop_map(sp, idx, coef)).max() < 1e-9 * np.abs(m1).max()
    d1 = O.direct_map(sc, fr)
    assert np.abs(d1 - ONP.direct_map(sc, fr)).max() < 1e-9 * np.abs(d1).max()


def test_hop_tracks_direct_within_cauchy_schwarz():
    # test_hopping.cpp:61-92 (Mc = 1)
    sc = S.small(scheme=S.POLY3, nx=12, ny=10)
    idx, coef, mres = O.build_table(sc)
    fr, _ = O.synth(sc, 1, 2)
    hop = O.hop_map(O.spectra(fr, sc.n_fft), idx, coef)
    direct = O.direct_map(sc, fr)
    for t in range(2):
        for b in range(0, sc.n_bins, 7):
            x = sc.grid_point(b)
            bound = 0.0
            for p in range(sc.n_pairs):
                r = O.sensed_range(sc.range_scale, sc.tx[p], sc.rx[p], x)
                a = np.exp(2j * np.pi * r * np.arange(sc.n_samples) / sc.n_samples)
                z = abs(np.sum(fr[t, p] * np.conj(a)))
                nrm = np.linalg.norm(fr[t, p])
                bound += 2 * z * mres * nrm + mres * mres * nrm * nrm
            assert abs(hop[t, b] - direct[t, b]) <= bound + 1e-9


def test_table_thread_invariance_and_window_error():
    sc = S.small(scheme=S.POLY3, nx=11, ny=9)
    a = O.build_table(sc, threads=1)
    b = O.build_table(sc, threads=4)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    with pytest.raises(O.OracleError, match=r"hop table: sensed range outside \[0, n_samples\)"):
        O.build_table(sc.with_(bandwidth=1e9), wrap=False)
    with pytest.raises(O.OracleError, match="scene outside unambiguous window"):
        O.synth(sc.with_(bandwidth=1e9), 0, 2, wrap=False)


def test_campaign_equals_map_argmax():
    sc = S.small(nx=14, ny=12)
    idx, coef, _ = O.build_table(sc)
    ei, ev = O.campaign_hop(sc, idx, coef, 5, 6, threads=2)
    fr, _ = O.synth(sc, 5, 6)
    m = O.hop_map(O.spectra(fr, sc.n_fft), idx, coef)
    assert np.array_equal(ei, np.argmax(m, axis=1))
    assert np.allclose(ev, m.max(axis=1))
    di, dv = O.campaign_direct(sc, 5, 6, threads=3)
    d = O.direct_map(sc, fr)
    assert np.array_equal(di, np.argmax(d, axis=1))


def test_topk_local_max():
    sc = S.small(nx=8, ny=6)
    m = np.zeros(sc.n_bins)
    m[9] = 5.0
    m[10] = 5.0  # plateau: smallest index wins
    m[40] = 7.0
    m[30] = 1.0
    idx, val = O.topk_local_max(sc, m, 4)
    assert list(idx[:3]) == [40, 9, 30]
    assert val[0] == 7.0


def test_golden_fixture_regression():
    f = np.load(GOLD / "small_c1like.npz")
    sc = S.small(**json.loads(str(f["scene_kw"])))
    idx, coef, _ = O.build_table(sc)
    assert np.array_equal(idx, f["idx"])
    assert np.abs(coef - f["coef"]).max() < 1e-12
    fr, truth = O.synth(sc, 0, int(f["trials"]))
    assert np.abs(fr - f["frames"]).max() < 1e-12
    m = O.hop_map(O.spectra(fr, sc.n_fft), idx, coef)
    assert np.abs(m - f["hop_map"]).max() < 1e-9 * np.abs(m).max()
    assert np.array_equal(np.argmax(m, axis=1), f["hop_argmax"])
    d = O.direct_map(sc, fr)
    assert np.array_equal(np.argmax(d, axis=1), f["direct_argmax"])
