"""Multi-GPU host logic: one process per GPU, torch.distributed for plumbing.

The hot path shards two ways:
  * trials: rank r owns a contiguous block of Monte-Carlo trials and
    synthesises them from (seed, trial) counters — no signal traffic; the
    only collective is one all-reduce(SUM) of a small statistics vector per
    campaign cell (hit_ratio / RMSE, src/montecarlo.cpp:181-216);
  * location grid (c5): every rank synthesises the same trials and scans its
    own slab of the grid; per-trial candidates merge with one
    all-reduce(MAX) of the 64-bit key  float_bits(value) << 32 | (2^32-1-bin),
    which orders by value then smallest bin (argmax_index tie rule,
    src/direct.cpp:55-62). Non-negative float bits keep the key below 2^63,
    so it travels as int64.
The same code runs over NCCL on GPUs and over gloo in the CPU tests.
"""
from __future__ import annotations

import numpy as np

STATS_FIELDS = ("count", "hits_1m", "sq_err_sum", "hits_half_res")


def shard(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) block of n items for rank (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def grid_slab(nz: int, ny: int, world: int, rank: int) -> tuple[int, int]:
    """Location-grid sharding: rank's [z0, z1) slab (or y rows for 2-D)."""
    return shard(nz if nz > 1 else ny, world, rank)


def campaign_stats(scene, est_idx: np.ndarray, truth: np.ndarray, threshold_m: float = 1.0) -> np.ndarray:
    """[count, hits within threshold, sum of squared location error, hits
    within half a range resolution] for single-target trials (truth [T, K, 3],
    target 0). Location of the estimate = its grid point."""
    est = scene.grid_points(est_idx)
    err = np.linalg.norm(est - truth[:, 0, :], axis=-1)
    half_res = 0.5 * scene.c / (2 * scene.bandwidth)
    return np.array([float(len(err)), float(np.sum(err <= threshold_m)), float(np.sum(err * err)),
                     float(np.sum(err <= half_res))])


def multi_target_stats(scene, est_idx: np.ndarray, truth: np.ndarray,
                       threshold_m: float = 1.0) -> np.ndarray:
    """K-target trials (BASELINE c3/c5): estimates [T, K] (bin, -1 = none)
    assigned to truths [T, K, 3] by the permutation of least total squared
    error (K <= 6: exhaustive). Returns the same 4-vector as campaign_stats,
    counted per target; a missing estimate counts as a miss at distance
    `miss_m` (the grid diagonal)."""
    import itertools
    T, K = est_idx.shape
    miss = float(np.linalg.norm(np.asarray(scene.grid_spacing) * np.asarray(scene.grid_n)))
    half_res = 0.5 * scene.c / (2 * scene.bandwidth)
    perms = list(itertools.permutations(range(K)))
    out = np.zeros(4)
    for t in range(T):
        pts = np.full((K, 3), np.nan)
        ok = est_idx[t] >= 0
        pts[ok] = scene.grid_points(est_idx[t][ok])
        d = np.linalg.norm(pts[:, None, :] - truth[t][None, :, :], axis=-1)
        d = np.where(np.isnan(d), miss, d)
        best = min(perms, key=lambda pm: sum(d[i, pm[i]] ** 2 for i in range(K)))
        err = np.array([d[i, best[i]] for i in range(K)])
        out += [K, np.sum(err <= threshold_m), np.sum(err * err), np.sum(err <= half_res)]
    return out


def summarize(stats: np.ndarray) -> dict:
    count = max(stats[0], 1.0)
    return {"trials": int(stats[0]), "hit_ratio_1m": stats[1] / count,
            "rmse_m": float(np.sqrt(stats[2] / count)), "hit_ratio_half_res": stats[3] / count}


def allreduce_stats(stats: np.ndarray, device=None) -> np.ndarray:
    """SUM over ranks (NCCL on GPU tensors, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(stats, dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def encode_keys(values: np.ndarray, bins: np.ndarray) -> np.ndarray:
    """Per-trial (value >= 0, global bin) -> int64 key, max == argmax rule."""
    vb = np.asarray(values, dtype=np.float32).view(np.uint32).astype(np.int64)
    return (vb << 32) | (0xFFFFFFFF - np.asarray(bins, dtype=np.int64))


def decode_keys(keys: np.ndarray):
    keys = np.asarray(keys, dtype=np.int64)
    bins = 0xFFFFFFFF - (keys & 0xFFFFFFFF)
    vals = (keys >> 32).astype(np.uint32).view(np.float32)
    return bins, vals


def allreduce_argmax(values: np.ndarray, bins: np.ndarray, device=None):
    """Merge per-rank shard winners into the global per-trial argmax."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(encode_keys(values, bins)).to(device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return decode_keys(t.cpu().numpy())


def max_over_ranks(x: float, device=None) -> float:
    """Step time of a multi-rank run: the slowest rank (max over ranks)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def merge_topk(bins: np.ndarray, values: np.ndarray, k: int):
    """Per-trial top-k over candidate lists from several shards: bins/values
    [S, T, k] (bin -1 = none) -> ([T, k], [T, k]) ranked by (value desc, bin
    asc), the order of the key above. Exact when every shard reports the k
    best local maxima of its core layers (halo shards) — a global top-k
    maximum is a core maximum of exactly one shard and ranks in its top-k."""
    bins = np.asarray(bins, dtype=np.int64)
    values = np.asarray(values, dtype=np.float32)
    S, T, kk = bins.shape
    keys = encode_keys(np.where(bins >= 0, values, 0.0), np.where(bins >= 0, bins, 0))
    keys = np.where(bins >= 0, keys, -1).transpose(1, 0, 2).reshape(T, S * kk)
    order = np.argsort(-keys, axis=1, kind="stable")[:, :k]
    top = np.take_along_axis(keys, order, axis=1)
    b, v = decode_keys(np.where(top >= 0, top, 0))
    return np.where(top >= 0, b, -1), np.where(top >= 0, v, 0.0).astype(np.float32)


def allgather_topk(bins: np.ndarray, values: np.ndarray, k: int, device=None):
    """The c5 multi-target exchange: one all-gather of every
    rank's k candidates per trial, then merge_topk on each rank."""
    import torch
    import torch.distributed as dist
    bins = np.asarray(bins, dtype=np.int64)
    values = np.asarray(values, dtype=np.float32)
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return merge_topk(bins[None], values[None], k)
    keys = encode_keys(np.where(bins >= 0, values, 0.0), np.where(bins >= 0, bins, 0))
    keys = np.where(bins >= 0, keys, -1)
    t = torch.from_numpy(keys).to(device)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    allk = np.stack([p.cpu().numpy() for p in parts])  # [S, T, k]
    b, v = decode_keys(np.where(allk >= 0, allk, 0))
    return merge_topk(np.where(allk >= 0, b, -1), v, k)
