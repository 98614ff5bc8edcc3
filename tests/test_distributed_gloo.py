"""CPU, world_size 2 over gloo: the N>1 host logic of the trial-sharded and
location-grid-sharded paths, with the fp64 oracle as the per-rank engine.

Checks the reference's determinism property lifted to ranks
(test_montecarlo.cpp:125-141: identical results for any thread count):
per-trial estimates and the all-reduced statistics equal the single-process
run, and the cross-shard argmax merge equals the full-grid argmax.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2307_16550_b200 import distributed as D
from paper_2307_16550_b200 import scene as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = S.small(nx=14, ny=12, scheme=S.POLY3)
        T = 23
        idx, coef, _ = O.build_table(sc)
        # trial sharding
        lo, hi = D.shard(T, world, rank)
        ei, ev = O.campaign_hop(sc, idx, coef, lo, hi - lo, threads=1)
        _, truth = O.synth(sc, lo, hi - lo)
        stats = D.allreduce_stats(D.campaign_stats(sc, ei, truth))
        # location-grid sharding: every rank the same trials, its own y-rows
        fr, _ = O.synth(sc, 0, 5)
        m = O.hop_map(O.spectra(fr, sc.n_fft), idx, coef)
        y0, y1 = D.grid_slab(1, sc.grid_n[1], world, rank)
        b0, b1 = y0 * sc.grid_n[0], y1 * sc.grid_n[0]
        loc = np.argmax(m[:, b0:b1], axis=1)
        bins, vals = D.allreduce_argmax(m[np.arange(5), b0 + loc], b0 + loc)
        tmax = D.max_over_ranks(float(rank + 1))
        out[rank] = (lo, hi, ei, stats, bins, tmax)
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_matches_single_process():
    from oracle import oracle as O
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    sc = S.small(nx=14, ny=12, scheme=S.POLY3)
    idx, coef, _ = O.build_table(sc)
    ei, _ = O.campaign_hop(sc, idx, coef, 0, 23, threads=1)
    _, truth = O.synth(sc, 0, 23)
    single = D.campaign_stats(sc, ei, truth)
    merged = np.concatenate([out[r][2] for r in range(world)])
    assert np.array_equal(merged, ei)
    for r in range(world):
        assert np.allclose(out[r][3], single)
        assert out[r][5] == 2.0
    fr, _ = O.synth(sc, 0, 5)
    m = O.hop_map(O.spectra(fr, sc.n_fft), idx, coef)
    assert np.array_equal(out[0][4], np.argmax(m, axis=1))
    assert np.array_equal(out[1][4], np.argmax(m, axis=1))


def test_shard_and_keys():
    assert [D.shard(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert D.shard(0, 2, 1) == (0, 0)
    vals = np.array([1.5, 1.5, 0.0, 3.0], dtype=np.float32)
    bins = np.array([7, 3, 0, 123456789])
    keys = D.encode_keys(vals, bins)
    assert (keys >= 0).all()
    b, v = D.decode_keys(keys)
    assert np.array_equal(b, bins) and np.array_equal(v, vals)
    # equal values: the smaller bin has the larger key
    assert keys[1] > keys[0]
    s = D.summarize(np.array([4.0, 2.0, 8.0, 1.0]))
    assert s["hit_ratio_1m"] == 0.5 and s["rmse_m"] == pytest.approx(np.sqrt(2.0))


def _core_topk(sub: np.ndarray, nx: int, core: slice, row0: int, k: int):
    """numpy restatement of the halo-shard pick: local maxima (> smaller-index
    neighbours, >= larger ones) of the core rows of a sub-map whose halo rows
    complete their neighbourhoods; k best by (value desc, bin asc)."""
    m = np.pad(sub.reshape(-1, nx), 1, constant_values=-np.inf)
    c = m[1:-1, 1:-1]
    small = np.maximum.reduce([m[:-2, :-2], m[:-2, 1:-1], m[:-2, 2:], m[1:-1, :-2]])
    large = np.maximum.reduce([m[1:-1, 2:], m[2:, :-2], m[2:, 1:-1], m[2:, 2:]])
    lm = (c > small) & (c >= large)
    lm[: core.start] = False
    lm[core.stop:] = False
    ys, xs = np.nonzero(lm)
    bins = (row0 + ys) * nx + xs
    vals = c[ys, xs].astype(np.float32)
    order = np.lexsort((bins, -vals))[:k]
    out_b = np.full(k, -1, dtype=np.int64)
    out_v = np.zeros(k, dtype=np.float32)
    out_b[: order.size], out_v[: order.size] = bins[order], vals[order]
    return out_b, out_v


def _topk_worker(rank, world, port, out):
    import torch.distributed as dist
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = S.small(n_targets=3, amp_mode=S.AMP_CGAUSS_PER_PAIR, snr_mode=S.SNR_UNIFORM_PER_PAIR,
                     snr_lo=5.0, snr_hi=20.0, nx=30, ny=26, scheme=S.NEAREST)
        T, K = 7, 3
        idx, coef, _ = O.build_table(sc)
        fr, _ = O.synth(sc, 0, T)
        m = O.hop_map(O.spectra(fr, sc.n_fft), idx, coef).astype(np.float32)
        nx, ny = sc.grid_n[0], sc.grid_n[1]
        y0, y1 = D.grid_slab(1, ny, world, rank)
        h0, h1 = max(0, y0 - 1), min(ny, y1 + 1)  # halo rows
        cand = [_core_topk(m[t, h0 * nx:h1 * nx], nx, slice(y0 - h0, y1 - h0), h0, K)
                for t in range(T)]
        bins = np.stack([c[0] for c in cand])
        vals = np.stack([c[1] for c in cand])
        out[rank] = D.allgather_topk(bins, vals, K)
    finally:
        dist.destroy_process_group()


def test_two_rank_halo_topk_merge_equals_full_grid():
    # c5-style location-grid sharding with K targets: halo shards report the
    # top-K maxima of their core rows, one all-gather merges them
    from oracle import oracle as O
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_topk_worker, args=(world, port, out), nprocs=world, join=True)
    sc = S.small(n_targets=3, amp_mode=S.AMP_CGAUSS_PER_PAIR, snr_mode=S.SNR_UNIFORM_PER_PAIR,
                 snr_lo=5.0, snr_hi=20.0, nx=30, ny=26, scheme=S.NEAREST)
    idx, coef, _ = O.build_table(sc)
    fr, _ = O.synth(sc, 0, 7)
    m = O.hop_map(O.spectra(fr, sc.n_fft), idx, coef).astype(np.float32).astype(np.float64)
    for t in range(7):
        ob, _ = O.topk_local_max(sc, m[t], 3)
        for r in range(world):
            assert np.array_equal(out[r][0][t], ob), (t, r, out[r][0][t], ob)


def test_merge_topk_orders_by_value_then_bin():
    b = np.array([[[5, 9, -1]], [[2, 7, 1]]])
    v = np.array([[[3.0, 1.0, 0.0]], [[3.0, 2.0, 0.5]]], dtype=np.float32)
    mb, mv = D.merge_topk(b, v, 3)
    assert mb.tolist() == [[2, 5, 7]] and mv.tolist() == [[3.0, 3.0, 2.0]]
