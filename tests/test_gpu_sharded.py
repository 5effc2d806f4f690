"""The multi-GPU code path (band sharding + exact two-step MIN merge + finalize) on real
hardware: two ranks share the one B200 of the pool, exchanging partials with the gloo
backend (a host-mediated collective: no kernel of one rank waits on the other). The
merged result must be bit-identical to the single-process run."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, t, lmin, lmax, out, mode="bands", backend="gloo"):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2008_13447_b200 import _lib, distributed, ingest
        s = ingest(t)
        sess = _lib.Session(0)
        if mode == "lengths":
            # NCCL: a 1-rank group with the exchange forced on, so the two all-reduces over
            # the library's device buffers run through NCCL on the B200
            distributed.profile_length_sharded(sess, s, lmin, lmax, rank, world,
                                               exchange=True if backend == "nccl" else None)
        else:
            distributed.profile_sharded(sess, s, lmin, lmax, rank, world)
        d, nm, ln, ix, pop = sess.valmp_arrays()
        off, nbr, dd = sess.smallest_rows(4)
        disc_d, disc_o = sess.discords(3)
        if rank == 0:
            np.savez(out, d=d, nm=nm, ln=ln, ix=ix, pop=pop, off=off, nbr=nbr, dd=dd,
                     disc_d=disc_d, disc_o=disc_o)
        sess.close()
    finally:
        dist.destroy_process_group()


def _sharded_equals_single(tmp_path, world, mode, t, lmin, lmax, backend="gloo"):
    import torch.multiprocessing as mp
    from paper_2008_13447_b200 import _lib, ingest
    out = str(tmp_path / f"sharded_{mode}_{world}_{backend}.npz")
    mp.start_processes(_rank, args=(world, _free_port(), t, lmin, lmax, out, mode, backend), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out)
    sess = _lib.session(0)
    with sess.lock:
        s = ingest(t)
        sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
        sess.profile(lmin, lmax)
        sess.finalize()
        ref = sess.valmp_arrays()
        rows = sess.smallest_rows(4)
        disc = sess.discords(3)
    for a, b in zip(ref, [got["d"], got["nm"], got["ln"], got["ix"], got["pop"]]):
        assert np.array_equal(a, b)
    for a, b in zip(rows, [got["off"], got["nbr"], got["dd"]]):
        assert np.array_equal(a, b)
    assert np.array_equal(disc[1], got["disc_o"]) and np.array_equal(disc[0], got["disc_d"])


def test_two_ranks_equal_single(tmp_path):
    """Band shards: bit-identical to one process."""
    t = np.cumsum(np.random.default_rng(44).standard_normal(6000))
    _sharded_equals_single(tmp_path, 2, "bands", t, 48, 64)


@pytest.mark.parametrize("world", [2, 3])
def test_length_shards_equal_single(tmp_path, world):
    """Length shards (each rank: seeds carried to its first length, a full-fold pass, then
    filtered lengths): bit-identical to one process."""
    t = np.cumsum(np.random.default_rng(45).standard_normal(6000))
    _sharded_equals_single(tmp_path, world, "lengths", t, 48, 64)


def test_nccl_exchange_single_rank(tmp_path):
    """The NCCL transport of the length-shard exchange (MIN / MAX all-reduce on the library's
    own device buffers via __cuda_array_interface__) on the pool's one GPU: a 1-rank NCCL
    group with the exchange forced on must reproduce the single-process run bit for bit."""
    t = np.cumsum(np.random.default_rng(31).standard_normal(20000))
    _sharded_equals_single(tmp_path, 1, "lengths", t, 100, 116, backend="nccl")
