"""GHT1 hop-table container and scene hash.

Reference: save_hop_table / load_hop_table (src/interp.cpp:225-389, format
include/gridhop/interp.hpp:69-77), scene_hash (src/model.cpp:135-166), and
their tests (tests/test_interp.cpp:208-293: exact round trip; stale,
truncated, bad-magic and missing files refused). The CPU tests run the
library's host-side container code on tables built by the oracle; the GPU
tests go through device tables (gh_table_save / gh_table_load).
"""
import struct

import numpy as np
import pytest

import paper_2307_16550_b200 as gh
from paper_2307_16550_b200 import scene as S
from oracle import oracle as O


def fnv1a_scene_hash(n_chirps, n_samples, f0, bandwidth, chirp_duration, tx, rx):
    """Independent restatement of model.cpp:135-166 (its offset basis
    1469598103934665603, prime 1099511628211, fields in order)."""
    h = 1469598103934665603
    data = struct.pack("<III", len(rx), n_chirps, n_samples)
    data += struct.pack("<ddd", f0, bandwidth, chirp_duration)
    data += struct.pack("<dd", *tx)
    for x, y in rx:
        data += struct.pack("<dd", x, y)
    for b in data:
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


RX = [[10.0, 0.0], [0.0, 10.0], [-10.0, 0.5]]


def test_scene_hash_matches_restatement_and_binds_constants():
    args = (16, 64, 77e9, 250e6, 20e-6, [0.0, 0.0], RX)
    h = gh.scene_hash(*args)
    assert h == fnv1a_scene_hash(*args)
    # test_interp.cpp:254-260: a shifted f0 or a moved receiver changes it
    assert gh.scene_hash(16, 64, 77e9 + 1e6, 250e6, 20e-6, [0.0, 0.0], RX) != h
    rx2 = [list(p) for p in RX]
    rx2[1][0] += 0.5
    assert gh.scene_hash(16, 64, 77e9, 250e6, 20e-6, [0.0, 0.0], rx2) != h


def _oracle_table(scheme):
    sc = S.small(scheme=scheme, nx=9, ny=7)
    idx, coef, mr = O.build_table(sc)
    return sc, idx, coef, mr


@pytest.mark.parametrize("scheme", [S.NEAREST, S.LINEAR, S.POLY3, S.POLAR])
def test_round_trip_is_exact(tmp_path, scheme):
    sc, idx, coef, mr = _oracle_table(scheme)
    path = tmp_path / "t.ght"
    gh.ght1_write(path, idx, coef, sc.os_range, sc.n_samples, 0x1234ABCD5678EF90, mr)
    hdr, idx2, coef2 = gh.ght1_read(path)
    assert hdr == {"n_pairs": sc.n_pairs, "n_bins": sc.n_bins, "k": idx.shape[2],
                   "os_range": sc.os_range, "n_samples": sc.n_samples,
                   "scene_hash": 0x1234ABCD5678EF90, "max_residual": mr}
    assert np.array_equal(idx2, idx)
    assert np.array_equal(coef2.view(np.float64), coef.view(np.float64))  # bit-exact doubles


def test_byte_layout_follows_the_reference(tmp_path):
    sc, idx, coef, mr = _oracle_table(S.LINEAR)
    path = tmp_path / "t.ght"
    gh.ght1_write(path, idx, coef, sc.os_range, sc.n_samples, 77, mr)
    raw = path.read_bytes()
    G, P, K = idx.shape
    assert raw[:4] == b"GHT1"
    assert struct.unpack_from("<6I", raw, 4) == (1, P, G, K, sc.os_range, sc.n_samples)
    assert struct.unpack_from("<Q", raw, 28)[0] == 77
    assert struct.unpack_from("<d", raw, 36)[0] == mr
    assert len(raw) == 44 + G * P * K * 20
    # first entry: K u32 indices, then K (re, im) f64 pairs (interp.cpp:306-314)
    assert list(struct.unpack_from(f"<{K}I", raw, 44)) == list(idx[0, 0])
    re_im = struct.unpack_from(f"<{2 * K}d", raw, 44 + 4 * K)
    assert np.array_equal(np.array(re_im[0::2]) + 1j * np.array(re_im[1::2]), coef[0, 0])


def test_corrupt_files_are_refused(tmp_path):
    sc, idx, coef, mr = _oracle_table(S.POLY3)
    path = tmp_path / "t.ght"
    gh.ght1_write(path, idx, coef, sc.os_range, sc.n_samples, 5, mr)
    raw = path.read_bytes()

    def expect(name, data, needle):
        p = tmp_path / name
        p.write_bytes(data)
        with pytest.raises(gh.GridhopRuntimeError, match=needle):
            gh.ght1_read(p)

    expect("short.ght", raw[: len(raw) // 2], "truncated")
    expect("tiny.ght", raw[:10], "truncated")
    expect("bad.ght", b"NOPE" + b" " * 40, "magic")
    expect("long.ght", raw + b"\0", "payload size mismatch")
    expect("ver.ght", raw[:4] + struct.pack("<I", 2) + raw[8:], "unsupported hop table version 2")
    expect("order.ght", raw[:16] + struct.pack("<I", 4) + raw[20:],
           "unsupported interpolation order 4")
    bad_idx = bytearray(raw)
    struct.pack_into("<I", bad_idx, 44, sc.n_fft)
    expect("idx.ght", bytes(bad_idx), "outside the FFT grid")
    with pytest.raises(gh.GridhopRuntimeError, match="cannot open"):
        gh.ght1_read(tmp_path / "missing.ght")


@pytest.mark.gpu
def test_device_table_save_load(tmp_path, ctx):
    sc = S.small(scheme=S.POLY3)
    t = gh.precompute_hop_table(ctx, sc)
    h = 0xFEEDFACE
    path = tmp_path / "dev.ght"
    gh.table_save(t, path, h)
    # the file is what the reference's loader reads: same operator as the oracle
    hdr, idx_f, coef_f = gh.ght1_read(path)
    oi, oc, _ = O.build_table(sc)
    assert np.array_equal(idx_f, oi)
    assert np.allclose(coef_f, oc, rtol=0, atol=1e-12)
    t2 = gh.table_load(ctx, path, sc, h)
    i1, c1 = t.download()
    i2, c2 = t2.download()
    assert np.array_equal(i1, i2) and np.array_equal(c1, c2)
    assert t2.max_residual == t.max_residual
    frames, _ = gh.synthesize(ctx, sc, 0, sc.trials)
    a1, v1 = gh.hop_argmax(ctx, t, frames)
    a2, v2 = gh.hop_argmax(ctx, t2, frames)
    assert np.array_equal(a1.cpu().numpy(), a2.cpu().numpy())
    assert np.array_equal(v1.cpu().numpy(), v2.cpu().numpy())


@pytest.mark.gpu
def test_device_load_refuses_stale_tables(tmp_path, ctx):
    sc = S.small(scheme=S.NEAREST)
    t = gh.precompute_hop_table(ctx, sc)
    path = tmp_path / "dev.ght"
    gh.table_save(t, path, 99)
    with pytest.raises(gh.GridhopRuntimeError, match="stale hop table"):
        gh.table_load(ctx, path, sc, 98)  # scene hash
    with pytest.raises(gh.GridhopRuntimeError, match="stale hop table"):
        gh.table_load(ctx, path, S.small(scheme=S.NEAREST, nx=23), 99)  # grid
    with pytest.raises(gh.GridhopRuntimeError, match="stale hop table"):
        gh.table_load(ctx, path, S.small(scheme=S.NEAREST, os=2), 99)  # oversampling
    shard = gh.precompute_hop_table_shard(ctx, sc, 0, 5)
    with pytest.raises(gh.InvalidArgument, match="shard"):
        gh.table_save(shard, tmp_path / "shard.ght", 99)
