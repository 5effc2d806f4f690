"""Two concurrent chains: on small series profile_impl walks the two halves of
the length range on two streams. Results must be bit-identical to the single chain, through
every entry point that runs phase 1, with and without the CUDA graph."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _all_profiles(run, lmin, lmax):
    return [run.profile(L) for L in range(lmin, lmax + 1)]


def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("graph", ["1", "0"])
def test_two_chains_equal_one_chain(graph):
    import paper_2008_13447_b200 as vl
    from paper_2008_13447_b200 import api, gen
    s = vl.ingest(gen.series_for(1))            # n = 4096
    lmin, lmax = 24, 72                         # 49 lengths

    def go():
        run = api.GpuRun(s, lmin, lmax)
        return run.stats, _all_profiles(run, lmin, lmax), run.valmp(), run.discords(2)

    st1, p1, v1, d1 = _with_env({"VLMP_CHAINS": "1", "VLMP_GRAPH": graph}, go)
    st2, p2, v2, d2 = _with_env({"VLMP_CHAINS": "2", "VLMP_GRAPH": graph}, go)
    assert st1["chains"] == 1 and st2["chains"] == 2
    for (mp_a, ip_a), (mp_b, ip_b) in zip(p1, p2):
        assert np.array_equal(ip_a, ip_b)
        assert np.array_equal(mp_a, mp_b, equal_nan=True)
    assert np.array_equal(v1.indices, v2.indices) and np.array_equal(v1.lengths, v2.lengths)
    assert np.array_equal(v1.distances, v2.distances, equal_nan=True)
    assert np.array_equal(d1[1], d2[1]) and np.array_equal(d1[0], d2[0], equal_nan=True)


def test_chains_default_and_short_ranges():
    """Automatic: two chains from 40 lengths on; shorter ranges and band shards stay one chain."""
    import paper_2008_13447_b200 as vl
    from paper_2008_13447_b200 import _lib, api, gen
    s = vl.ingest(gen.series_for(1))
    os.environ.pop("VLMP_CHAINS", None)
    assert api.GpuRun(s, 24, 72).stats["chains"] == 2
    assert api.GpuRun(s, 32, 64).stats["chains"] == 1
    sess = _lib.session(0)
    with sess.lock:
        sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
        sess.profile(24, 72, 0, 2, 0)            # a band shard
        sess.finalize()
        assert sess.stats()["chains"] == 1


def test_two_chains_against_oracle_with_flat_stretches():
    """The second chain starts like a length shard (direct-sum seeds, sampled folds): neighbours
    against the CPU oracle on a series with constant stretches and a wide variance range."""
    import paper_2008_13447_b200 as vl
    from paper_2008_13447_b200 import api
    from oracle import oracle
    rng = np.random.default_rng(11)
    t = np.cumsum(rng.standard_normal(3000))
    t[700:760] = t[700]
    t[1500:1800] *= 1e-3
    s = vl.ingest(t)
    lmin, lmax = 20, 44                         # 25 lengths: forced (VLMP_CHAINS=2 applies from 16 on)
    run = _with_env({"VLMP_CHAINS": "2"}, lambda: api.GpuRun(s, lmin, lmax))
    assert run.stats["chains"] == 2
    ref = oracle.run(s, lmin, lmax, keep_profiles=True)
    for L in range(lmin, lmax + 1):
        mp, ip = run.profile(L)
        omp, oip = ref["profiles"][L]
        fin = np.isfinite(omp)
        # ties within the key resolution may pick another neighbour of equal distance
        same = ip == oip
        assert np.allclose(mp[fin], omp[fin], atol=1e-7), L
        with np.errstate(invalid="ignore"):
            assert np.all(same | ~fin | (np.abs(mp - omp) < 1e-9)), L


def test_log_overflow_redo_with_two_chains(monkeypatch):
    """A run log too small for a length (VLMP_LOG_CAP test hook) in either chain: the run is
    redone exactly (one chain, FP64 filter path) and equals the normal result."""
    import paper_2008_13447_b200 as vl
    from paper_2008_13447_b200 import api
    s = vl.ingest(np.cumsum(np.random.default_rng(23).standard_normal(3000)))
    lmin, lmax = 32, 56
    monkeypatch.setenv("VLMP_CHAINS", "2")
    ref = api.GpuRun(s, lmin, lmax)
    assert ref.stats["chains"] == 2 and ref.stats["exact_redo"] == 0
    want = _all_profiles(ref, lmin, lmax)
    monkeypatch.setenv("VLMP_LOG_CAP", "16")
    run = api.GpuRun(s, lmin, lmax)
    assert run.stats["exact_redo"] >= 1
    for (mp, ip), (gmp, gip) in zip(want, _all_profiles(run, lmin, lmax)):
        assert np.array_equal(gip, ip) and np.array_equal(gmp, mp, equal_nan=True)
    monkeypatch.delenv("VLMP_LOG_CAP")
    again = api.GpuRun(s, lmin, lmax)              # and the session recovers its two-chain graph
    assert again.stats["chains"] == 2 and again.stats["exact_redo"] == 0
    for (mp, ip), (gmp, gip) in zip(want, _all_profiles(again, lmin, lmax)):
        assert np.array_equal(gip, ip) and np.array_equal(gmp, mp, equal_nan=True)
