"""MRF1 capture replay and multi-chirp frames.

Reference: write_frames / read_frames (src/frame_io.cpp:53-164, format
include/gridhop/frame_io.hpp:10-16) and their tests (tests/test_frame_io.cpp:
72-152: bit-exact round trip, empty capture legal, bad magic / version /
truncation / payload size named); scan_planes over Mc chirps
(src/hopping.cpp:59-117) for the replayed frames, checked against the
oracle's multi-chirp restatement.
"""
import struct

import numpy as np
import pytest

import paper_2307_16550_b200 as gh
from paper_2307_16550_b200 import scene as S
from oracle import oracle as O

TX = (0.13, -0.21)  # off the location grid (a station on a bin is degenerate)
RX = [[10.0, 0.0], [-4.0, 9.0]]


def _capture(T=3, Q=2, Mc=8, Ms=16, seed=101):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((T, Q, Mc, Ms)) + 1j * rng.standard_normal((T, Q, Mc, Ms))


def test_round_trip_bit_exact(tmp_path):
    fr = _capture()
    p = tmp_path / "cap.mrf"
    gh.mrf1_write(p, fr, 24e9, 250e6, 128e-6, TX, RX)
    hdr, rx, back = gh.mrf1_read(p)
    assert hdr == {"n_rx": 2, "n_chirps": 8, "n_samples": 16, "n_frames": 3, "f0": 24e9,
                   "bandwidth": 250e6, "chirp_duration": 128e-6, "tx": TX}
    assert np.array_equal(rx, np.array(RX))
    assert np.array_equal(back.view(np.float64), fr.view(np.float64))


def test_byte_layout(tmp_path):
    fr = _capture(T=2)
    p = tmp_path / "cap.mrf"
    gh.mrf1_write(p, fr, 24e9, 250e6, 128e-6, TX, RX)
    raw = p.read_bytes()
    assert raw[:4] == b"MRF1"
    assert struct.unpack_from("<5I", raw, 4) == (1, 2, 8, 16, 2)
    assert struct.unpack_from("<3d", raw, 24) == (24e9, 250e6, 128e-6)
    assert struct.unpack_from("<6d", raw, 48) == (*TX, 10.0, 0.0, -4.0, 9.0)
    # frames receiver-major, rows (chirps) row-major, (re, im) f64 pairs
    first = struct.unpack_from("<4d", raw, 96)
    assert first == (fr[0, 0, 0, 0].real, fr[0, 0, 0, 0].imag,
                     fr[0, 0, 0, 1].real, fr[0, 0, 0, 1].imag)
    assert len(raw) == 96 + fr.size * 16


def test_empty_capture_is_legal(tmp_path):
    p = tmp_path / "empty.mrf"
    gh.mrf1_write(p, np.zeros((0, 2, 8, 16), dtype=np.complex128), 24e9, 250e6, 128e-6, TX, RX)
    hdr, _, fr = gh.mrf1_read(p)
    assert hdr["n_frames"] == 0 and fr.shape == (0, 2, 8, 16) and hdr["n_chirps"] == 8


def test_bad_files_are_named(tmp_path):
    good = tmp_path / "good.mrf"
    gh.mrf1_write(good, _capture(T=2), 24e9, 250e6, 128e-6, TX, RX)
    raw = good.read_bytes()

    def expect(name, data, needle):
        p = tmp_path / name
        p.write_bytes(data)
        with pytest.raises(gh.GridhopRuntimeError, match=needle):
            gh.mrf1_read(p)

    expect("magic.mrf", b"XXXX" + raw[4:], "bad magic")
    v2 = bytearray(raw)
    v2[4] = 9
    expect("version.mrf", bytes(v2), "unsupported capture version")
    expect("trunc.mrf", raw[:30], "truncated")
    expect("short.mrf", raw[:-16], "payload size mismatch")
    expect("long.mrf", raw + b"\0" * 8, "payload size mismatch")
    with pytest.raises(gh.GridhopRuntimeError, match="cannot open"):
        gh.mrf1_read(tmp_path / "nope.mrf")


def test_writer_validates_like_the_reference(tmp_path):
    p = tmp_path / "x.mrf"
    with pytest.raises(gh.InvalidArgument, match="n_chirps must be >= 2"):
        gh.mrf1_write(p, _capture(Mc=1), 24e9, 250e6, 128e-6, TX, RX)
    with pytest.raises(gh.InvalidArgument, match="receivers coincide"):
        gh.mrf1_write(p, _capture(), 24e9, 250e6, 128e-6, TX, [[1.0, 1.0], [1.0, 1.0]])
    with pytest.raises(gh.InvalidArgument, match="receiver coincides with TX"):
        gh.mrf1_write(p, _capture(), 24e9, 250e6, 128e-6, TX, [list(TX), [1.0, 1.0]])
    with pytest.raises(gh.InvalidArgument, match="frame/receiver count mismatch"):
        gh.mrf1_write(p, _capture(Q=3), 24e9, 250e6, 128e-6, TX, RX)


def _capture_scene(hdr, rx, nx=21, ny=17, spacing=0.5, os=4):
    """The capture's geometry as TX-RX pairs (one TX, every RX), z = 0."""
    Q = hdr["n_rx"]
    tx = np.tile(np.array([[hdr["tx"][0], hdr["tx"][1], 0.0]]), (Q, 1))
    rx3 = np.column_stack([rx, np.zeros(Q)])
    ox, oy = -spacing * (nx - 1) / 2, -spacing * (ny - 1) / 2
    return S.Scene(name="capture", n_samples=hdr["n_samples"], os_range=os,
                   bandwidth=hdr["bandwidth"], tx=tx, rx=rx3, grid_origin=(ox, oy, 0.0),
                   grid_spacing=(spacing, spacing, 1.0), grid_n=(nx, ny, 1), scheme=S.NEAREST,
                   wrap=True)


def _synthetic_capture(sc, T, Mc, seed=7):
    """Targets at grid points, a Doppler phase ramp over chirps, CN noise."""
    rng = np.random.default_rng(seed)
    n = np.arange(sc.n_samples)
    fr = np.zeros((T, sc.n_pairs, Mc, sc.n_samples), dtype=np.complex128)
    pts = sc.grid_points(rng.integers(0, sc.n_bins, T))
    for t in range(T):
        for q in range(sc.n_pairs):
            r = sc.range_scale * (np.linalg.norm(pts[t] - sc.tx[q]) + np.linalg.norm(pts[t] - sc.rx[q]))
            u = rng.uniform(-2, 2)
            fr[t, q] = (np.exp(2j * np.pi * u * np.arange(Mc) / Mc)[:, None]
                        * np.exp(2j * np.pi * r * n / sc.n_samples)[None, :])
    fr += 0.3 * (rng.standard_normal(fr.shape) + 1j * rng.standard_normal(fr.shape))
    return fr


@pytest.mark.gpu
@pytest.mark.parametrize("Mc", [1, 4, 13])
def test_multi_chirp_hop_map_matches_oracle(ctx, Mc):
    sc = _capture_scene({"n_rx": 2, "n_samples": 64, "bandwidth": 250e6, "tx": TX}, np.array(RX))
    T = 21
    fr = _synthetic_capture(sc, T, Mc)
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map_mc(O.spectra(fr, sc.n_fft), oi, oc)
    import torch
    fd = torch.from_numpy(fr.astype(np.complex64)).cuda()
    t = gh.precompute_hop_table(ctx, sc)
    m = gh.hop_map_mc(ctx, t, fd).cpu().numpy()
    err = (np.abs(m - ref).max(axis=1) / np.abs(ref).max(axis=1)).max()
    assert err < 1e-4
    idx, _ = gh.hop_argmax_mc(ctx, t, fd)
    idx = idx.cpu().numpy()
    for i in range(T):
        a = int(np.argmax(ref[i]))
        if a != idx[i]:
            assert abs(ref[i][a] - ref[i][idx[i]]) <= 1e-5 * ref[i].max()
    if Mc == 1:  # the single-chirp path gives the same answers
        i1, _ = gh.hop_argmax(ctx, t, fd[:, :, 0, :].contiguous())
        assert np.array_equal(i1.cpu().numpy(), idx)


@pytest.mark.gpu
def test_capture_replay(ctx, tmp_path):
    # write a capture, read it back, rebuild the scene from its header and
    # estimate every frame's location through the multi-chirp hop path
    base = _capture_scene({"n_rx": 2, "n_samples": 64, "bandwidth": 250e6, "tx": TX}, np.array(RX))
    fr = _synthetic_capture(base, 9, 8, seed=3)
    p = tmp_path / "replay.mrf"
    gh.mrf1_write(p, fr, 24e9, 250e6, 128e-6, TX, RX)
    hdr, rx, back = gh.mrf1_read(p)
    sc = _capture_scene(hdr, rx)
    t = gh.precompute_hop_table(ctx, sc)
    import torch
    idx, _ = gh.hop_argmax_mc(ctx, t, torch.from_numpy(back.astype(np.complex64)).cuda())
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map_mc(O.spectra(back, sc.n_fft), oi, oc)
    assert np.array_equal(idx.cpu().numpy(), np.argmax(ref, axis=1))
    with pytest.raises(gh.InvalidArgument, match="K = 1"):
        t3 = gh.precompute_hop_table(ctx, sc, scheme=S.POLY3)
        gh.hop_argmax_mc(ctx, t3, torch.from_numpy(back.astype(np.complex64)).cuda())
