"""The N>1 path on CPU: world_size-2 gloo processes shard the diagonal bands,
compute band-restricted partial minima (oracle arithmetic), and merge them with
the same two-step exact MIN protocol the GPU ranks use over NCCL
(distributed.merge_partials). The merged result must equal the unsharded one,
including smallest-index tie-breaks."""

import os
import socket

import numpy as np
import pytest

from paper_2008_13447_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partials(t, lmin, lmax, bands, quantize):
    """Per (length, offset) min over cells whose diagonal lies in `bands`:
    key = bits of the (optionally quantised, to force ties) distance."""
    n = t.shape[0]
    A = n
    keys = np.full((lmax - lmin + 1) * A, np.float64(np.inf).view(np.int64), dtype=np.int64)
    idx = np.full(keys.shape, D.IDX_NONE, dtype=np.int64)
    d_lo = D.dlo(lmin) + bands[0] * D.BAND
    d_hi = D.dlo(lmin) + bands[1] * D.BAND
    for li, m in enumerate(range(lmin, lmax + 1)):
        w = np.lib.stride_tricks.sliding_window_view(t, m)
        z = (w - w.mean(1, keepdims=True)) / w.std(1, keepdims=True)
        dist = np.sqrt(np.maximum(((z[:, None, :] - z[None, :, :]) ** 2).sum(-1), 0))
        if quantize:
            dist = np.round(dist, 1)
        N = w.shape[0]
        e = (m + 1) // 2
        for i in range(N):
            for j in range(i + max(e, d_lo), min(N, i + d_hi)):
                k = np.float64(dist[i, j]).view(np.int64)
                for o, nb in ((i, j), (j, i)):
                    q = li * A + o
                    if (k, nb) < (keys[q], idx[q]):
                        keys[q], idx[q] = k, nb
    return keys, idx


def _worker(rank, world, port, t, lmin, lmax, quantize, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nb = D.n_bands(t.shape[0], lmin)
        cuts = D.band_split(t.shape[0], lmin, lmax, world)
        assert cuts[-1] == nb
        k, i = _partials(t, lmin, lmax, (cuts[rank], cuts[rank + 1]), quantize)
        kt, it = torch.from_numpy(k), torch.from_numpy(i)
        D.merge_partials(kt, it)
        if rank == 0:
            np.save(out + "_k.npy", kt.numpy())
            np.save(out + "_i.npy", it.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("quantize", [False, True])
def test_two_rank_merge_equals_single(tmp_path, quantize):
    import torch.multiprocessing as mp
    t = np.cumsum(np.random.default_rng(5).standard_normal(700))
    lmin, lmax = 8, 10
    out = str(tmp_path / "merged")
    mp.start_processes(_worker, args=(2, _free_port(), t, lmin, lmax, quantize, out),
                       nprocs=2, join=True, start_method="fork")
    nb = D.n_bands(t.shape[0], lmin)
    k1, i1 = _partials(t, lmin, lmax, (0, nb), quantize)
    assert np.array_equal(np.load(out + "_k.npy"), k1)
    assert np.array_equal(np.load(out + "_i.npy"), i1)


def _slab_worker(rank, world, port, n, lmin, lmax, stride, out):
    """Each rank owns the lengths length_split gives it: it fills only its slab (the value a
    rank computes for (li, o) is a function of (li, o) alone) and the all-gather must leave
    every rank with the complete buffer (int32 and float64, as the MP / IP buffers)."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cuts = D.length_split(n, lmin, lmax, world)
        nl = lmax - lmin + 1
        full = (np.arange(nl * stride, dtype=np.float64) * 1.5 - 7.0)
        for dtype in (torch.float64, torch.int32):
            buf = torch.full((nl * stride,), -1, dtype=dtype)
            a, b = int(cuts[rank]) * stride, int(cuts[rank + 1]) * stride
            buf[a:b] = torch.from_numpy(full[a:b]).to(dtype)
            D.gather_owned_slabs(buf, cuts, stride, rank, world)
            assert torch.equal(buf, torch.from_numpy(full).to(dtype)), (rank, dtype)
        if rank == 0:
            np.save(out, cuts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_length_slab_all_gather(tmp_path, world):
    """The length-shard exchange (distributed.gather_owned_slabs) on world-size 2 and 3 gloo
    groups: unequal slabs (work-balanced length cuts), padded all-gather, in-place scatter."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "cuts.npy")
    mp.start_processes(_slab_worker, args=(world, _free_port(), 65536, 256, 384, 37, out),
                       nprocs=world, join=True, start_method="fork")
    cuts = np.load(out)
    assert cuts[0] == 0 and cuts[-1] == 129 and np.all(np.diff(cuts) > 0)
