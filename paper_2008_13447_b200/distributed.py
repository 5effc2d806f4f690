"""Multi-GPU sharding: one process per GPU.

Length shards (default, `profile_length_sharded`). Each rank owns a contiguous run of
lengths of equal work and computes the complete profile of those lengths on its GPU, with
no exchange while it runs: its tile seeds are centred direct sums at its first length (the
FP32 walk only gates; every key comes from the exact FP64 runs), that length takes its
bounds from full folds over a sample of its bands, and every length then runs the FP32 walk
+ exact runs. Every length's whole triangle runs on one GPU, so every GPU stays fully
occupied at any world size. Each (length, offset) has exactly one owner, so the exchange is
an all-gather of each rank's finalized slab (`gather_owned_slabs`); the neighbours equal a
single run's (keys of a run may differ in their last bits where the run starts elsewhere,
which only matters at ties within ~1e-15; the GPU tests compare bit for bit).

Band shards (`profile_sharded`), kept for very long lengths ranges per GPU:

Partition. The pair triangle at length l holds cells (i, i+d), d >= ceil(l/2).
Bands of 256 consecutive diagonals are the unit (one warp tile wide); band b's
work summed over lengths is sum_l sum_{d in b, d >= e_l} (N_l - d)_+ (closed
form per length). Ranks get contiguous band ranges of equal cumulative work
(SURVEY.md §8(e)). No data moves between ranks during the scan: each rank's
filter bound comes from its own previous-length winners (any valid cell value is
an upper bound on the global minimum, so rank-local bounds stay exact).

Exchange. Per (length, offset) every rank holds (key, idx): key = order-
preserving uint64 bits of the clamped r' = 1 - corr (+inf bits = none), idx =
neighbour. The lexicographic (key, smallest idx) rule of profile.py:308 is
realised as: all-reduce MIN over keys; idx := INT64_MAX where the local key
differs from the merged key; all-reduce MIN over idx. Keys are non-negative
doubles, so their bit patterns order correctly as int64.
"""

from __future__ import annotations

import numpy as np

BAND = 256   # = 32 * VLMP_D of libvlmp (diagonals per warp tile)
IDX_NONE = np.iinfo(np.int64).max


def dlo(lmin: int) -> int:
    return (lmin + 1) // 2


def n_bands(n: int, lmin: int) -> int:
    N = n - lmin + 1
    span = N - dlo(lmin)
    return (span + BAND - 1) // BAND if span > 0 else 0


def band_work(n: int, lmin: int, lmax: int, b: int) -> float:
    d_lo = dlo(lmin) + b * BAND
    d_hi = d_lo + BAND
    w = 0.0
    for m in range(lmin, lmax + 1):
        N = n - m + 1
        lo, hi = max(d_lo, (m + 1) // 2), min(d_hi, N)
        if hi > lo:
            w += (hi - lo) * N - (lo + hi - 1) * (hi - lo) / 2.0
    return w


def band_split(n: int, lmin: int, lmax: int, parts: int) -> np.ndarray:
    """Contiguous band cuts with equal cumulative work (same rule as vlmp_band_split)."""
    nb = n_bands(n, lmin)
    w = np.array([band_work(n, lmin, lmax, b) for b in range(nb)])
    tot = w.sum()
    cuts = np.zeros(parts + 1, dtype=np.int64)
    acc, b = 0.0, 0
    for p in range(1, parts):
        target = tot * p / parts
        while b < nb and acc + w[b] <= target:
            acc += w[b]
            b += 1
        cuts[p] = b
    cuts[parts] = nb
    return cuts


def length_work(n: int, m: int) -> float:
    """Non-trivial pairs at length m: (N - e)(N - e + 1) / 2."""
    k = (n - m + 1) - (m + 1) // 2
    return k * (k + 1) / 2.0 if k > 0 else 0.0


# a shard's first length folds (a sample of) its bands for bounds, then runs the FP32 pass:
# ~2.5x a filtered length (config 2: 1.57 ms vs 0.62 ms)
FULL_PASS_FACTOR = 2.5


def length_split(n: int, lmin: int, lmax: int, parts: int) -> np.ndarray:
    """Contiguous length-index cuts [c_r, c_{r+1}) of [0, lmax - lmin + 1) with equal work,
    each shard's first (full-fold) length counted at FULL_PASS_FACTOR; cuts are placed at
    the nearest length boundary. More shards than lengths leave the extra shards empty."""
    nl = lmax - lmin + 1
    w = np.array([length_work(n, lmin + li) for li in range(nl)])
    extra = (FULL_PASS_FACTOR - 1.0) * (w.mean() if nl else 0.0)
    live = max(1, min(parts, nl))
    target = (w.sum() + live * extra) / live
    cuts = [0]
    acc = extra
    for li in range(nl):
        if len(cuts) < live and li > cuts[-1] and acc + w[li] / 2.0 > target \
                and nl - li >= live - len(cuts):
            cuts.append(li)
            acc = extra
        acc += w[li]
    while len(cuts) < live:
        cuts.append(cuts[-1] + 1)
    cuts += [nl] * (parts + 1 - len(cuts))
    return np.array(cuts, dtype=np.int64)


def merge_partials(keys, idx, group=None):
    """Exact (key, smallest idx) merge of torch int64 tensors across the group,
    in place. Works for any backend (NCCL on GPU tensors, gloo on CPU tensors)."""
    import torch
    import torch.distributed as dist
    merged = keys.clone()
    dist.all_reduce(merged, op=dist.ReduceOp.MIN, group=group)
    idx.masked_fill_(keys != merged, IDX_NONE)
    dist.all_reduce(idx, op=dist.ReduceOp.MIN, group=group)
    keys.copy_(merged)
    return keys, idx


def _exchange_and_finalize(sess, rank, world, group):
    import torch
    with sess.lock:
        n_len, stride = sess.partials_size()
        dev = torch.device("cuda", sess.device)
        keys = torch.empty(n_len * stride, dtype=torch.int64, device=dev)
        idx = torch.empty(n_len * stride, dtype=torch.int64, device=dev)
        sess.partials_export(keys.data_ptr(), idx.data_ptr())
    if world > 1:
        import torch.distributed as dist
        merged = keys.clone()
        dist.all_reduce(merged, op=dist.ReduceOp.MIN, group=group)
        torch.cuda.synchronize(dev)
        with sess.lock:
            sess.partials_mask_idx(merged.data_ptr(), keys.data_ptr(), idx.data_ptr())
        dist.all_reduce(idx, op=dist.ReduceOp.MIN, group=group)
        torch.cuda.synchronize(dev)
        keys = merged
    with sess.lock:
        sess.partials_import(keys.data_ptr(), idx.data_ptr())
        sess.finalize()


class _DeviceArray:
    """__cuda_array_interface__ view of a library-owned device buffer (no copy)."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def gather_owned_slabs(buf, cuts, stride: int, rank: int, world: int, group=None):
    """Every (length, offset) has exactly one owner rank, so the exchange is an all-gather of
    each rank's contiguous slab of lengths [cuts[r], cuts[r+1]) of ``buf`` ([n_len * stride],
    a torch view of the library's device buffer), in place. Slabs are padded to the largest
    shard so one all_gather_into_tensor moves them (NCCL over NVLink); this moves each rank's
    bytes once, half the ring traffic of an all-reduce over the whole buffer. Backends without
    CUDA all-gather (gloo) go through host memory."""
    import torch
    import torch.distributed as dist
    rows = [int(cuts[r + 1] - cuts[r]) for r in range(world)]
    slab = max(rows) * stride
    lo = int(cuts[rank]) * stride
    send = torch.zeros(slab, dtype=buf.dtype, device=buf.device)
    send[:rows[rank] * stride].copy_(buf[lo:lo + rows[rank] * stride])
    cpu = dist.get_backend(group) == "gloo"
    if cpu:
        send = send.cpu()
    out = torch.empty(world * slab, dtype=buf.dtype, device=send.device)
    if cpu:
        dist.all_gather(list(out.chunk(world)), send, group=group)
    else:
        dist.all_gather_into_tensor(out, send, group=group)
    for r in range(world):
        if r != rank and rows[r]:
            a = int(cuts[r]) * stride
            buf[a:a + rows[r] * stride].copy_(out[r * slab:r * slab + rows[r] * stride])
    return buf


def profile_length_sharded(sess, series, lmin: int, lmax: int, rank: int, world: int, group=None,
                           upload: bool = True, exchange: bool | None = None):
    """This rank's lengths on its session's device, finalized there; the per-length profile
    values (MP double, IP int32) are then all-gathered slab by slab across ranks (every
    (length, offset) is owned by exactly one rank) and every rank builds the read-offs.
    ``upload=False`` reuses the series already resident on the device; ``exchange`` forces
    the collective step on (a 1-rank group still runs it) or off (default: world > 1)."""
    import torch
    cuts = length_split(series.n, lmin, lmax, world)
    lo, hi = int(cuts[rank]), int(cuts[rank + 1]) - 1
    with sess.lock:
        if upload:
            sess.set_series(series.values, series._cum, series._cum2, series.sigma_floor)
        # an empty shard (more ranks than lengths) still joins with neutral values
        sess.profile_lengths(lmin, lmax, lo, hi)
        sess.finalize_lengths(lo, hi)
    if (world > 1) if exchange is None else exchange:
        mp_ptr, ip_ptr, n_len, stride = sess.final_buffers()
        dev = torch.device("cuda", sess.device)
        mp = torch.as_tensor(_DeviceArray(mp_ptr, n_len * stride, "<f8"), device=dev)
        ip = torch.as_tensor(_DeviceArray(ip_ptr, n_len * stride, "<i4"), device=dev)
        gather_owned_slabs(mp, cuts, stride, rank, world, group)
        gather_owned_slabs(ip, cuts, stride, rank, world, group)
        torch.cuda.synchronize(dev)
    with sess.lock:
        sess.finalize_readoffs()
    return cuts


def profile_sharded(sess, series, lmin: int, lmax: int, rank: int, world: int, group=None,
                    upload: bool = True):
    """Run this rank's bands on its session's device, merge with the group and finalize.
    ``upload=False`` reuses the series already resident on the device."""
    import torch
    cuts = band_split(series.n, lmin, lmax, world)
    with sess.lock:
        if upload:
            sess.set_series(series.values, series._cum, series._cum2, series.sigma_floor)
        sess.profile(lmin, lmax, int(cuts[rank]), int(cuts[rank + 1]), 0)
        n_len, stride = sess.partials_size()
        dev = torch.device("cuda", sess.device)
        keys = torch.empty(n_len * stride, dtype=torch.int64, device=dev)
        idx = torch.empty(n_len * stride, dtype=torch.int64, device=dev)
        sess.partials_export(keys.data_ptr(), idx.data_ptr())
    if world > 1:
        import torch.distributed as dist
        merged = keys.clone()
        dist.all_reduce(merged, op=dist.ReduceOp.MIN, group=group)
        torch.cuda.synchronize(dev)
        with sess.lock:
            sess.partials_mask_idx(merged.data_ptr(), keys.data_ptr(), idx.data_ptr())
        dist.all_reduce(idx, op=dist.ReduceOp.MIN, group=group)
        torch.cuda.synchronize(dev)
        keys = merged
    with sess.lock:
        sess.partials_import(keys.data_ptr(), idx.data_ptr())
        sess.finalize()
    return cuts
