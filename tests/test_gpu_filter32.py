"""The FP32 filter walk (filter32.cu) against the FP64 filter (profile.cu k_tile<false>) and the
oracle. The FP32 walk decides only which cells reach the exact FP64 evaluation, under a
rigorous error slack, so every profile must equal the FP64 path's and the oracle's."""

import numpy as np
import pytest

import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import _lib, api, gen
from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _device():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    _lib.load()


def _both(s, lmin, lmax):
    a = api.GpuRun(s, lmin, lmax)
    pa = [a.profile(L) for L in range(lmin, lmax + 1)]
    sa = dict(a.stats)
    b = api.GpuRun(s, lmin, lmax, flags=_lib.FLAG_FP64_FILTER)
    pb = [b.profile(L) for L in range(lmin, lmax + 1)]
    assert b.stats["fp32_walk"] == 0
    return sa, pa, pb


def _planted(n, m, seed):
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.standard_normal(n))
    pat = np.cumsum(rng.standard_normal(m))
    for off in (n // 7, n // 2 + 11):
        t[off:off + m] = pat + rng.normal(0, 0.05, m) + t[off]
    return t


@pytest.mark.parametrize("case", ["cfg1", "planted", "sines", "small_walk0", "small_planted3"])
def test_fp32_walk_equals_fp64_filter(case):
    if case == "cfg1":
        t, lmin, lmax = gen.series_for(1), 32, 64
    elif case == "planted":
        t, lmin, lmax = _planted(24000, 200, 3), 150, 190
    elif case == "sines":
        x = np.arange(30000)
        t = np.sin(2 * np.pi * x / 173) + 0.6 * np.sin(2 * np.pi * x / 611) \
            + np.random.default_rng(4).normal(0, 0.2, x.size)
        lmin, lmax = 180, 200
    else:
        g = load_golden(case)
        t, lmin, lmax = g["t"], int(g["lmin"]), int(g["lmax"])
    sa, pa, pb = _both(vl.ingest(t), lmin, lmax)
    if len(t) >= 20000:   # long enough for the sampled start + filtered lengths on the FP32 walk
        assert sa["fp32_walk"] == 1 and sa["exact_redo"] == 0
        assert sa["run_cells"] > 0
    for L, (a, b) in zip(range(lmin, lmax + 1), zip(pa, pb)):
        assert np.array_equal(a[1], b[1]), L
        assert np.array_equal(a[0], b[0]), L


def test_fp32_buffers_follow_the_series():
    """A session that ran a short series must grow its FP32 buffers for a longer one."""
    api.GpuRun(vl.ingest(gen.series_for(1)), 32, 40)
    s = vl.ingest(_planted(40000, 120, 9))
    run = api.GpuRun(s, 100, 110)
    assert run.stats["fp32_walk"] == 1 and run.stats["exact_redo"] == 0


def _brute_refstats(s, L):
    """Nearest neighbours with the reference's window statistics (prefix sums, series.py:91-100)
    but exact centred co-moments (explicit window products, no recurrence): the arithmetic the
    drop-in's keys follow, without the recurrence error the reference engine adds."""
    t = s.values
    W = np.lib.stride_tricks.sliding_window_view(t, L)
    mu = (s._cum[L:] - s._cum[:-L]) / L
    var = np.maximum((s._cum2[L:] - s._cum2[:-L]) / L - mu * mu, 0.0)
    X = (W - mu[:, None]) / np.sqrt(var * L)[:, None]
    N, e = W.shape[0], (L + 1) // 2
    d = np.empty(N); nn = np.empty(N, dtype=np.int64)
    idx = np.arange(N)
    for b0 in range(0, N, 1024):
        r2 = np.maximum(2 * L * (1 - X[b0:b0 + 1024] @ X.T), 0)
        r2[np.abs(idx[b0:b0 + 1024, None] - idx[None, :]) < e] = np.inf
        nn[b0:b0 + 1024] = np.argmin(r2, 1)
        d[b0:b0 + 1024] = np.sqrt(r2[np.arange(r2.shape[0]), nn[b0:b0 + 1024]])
    pair = lambda a, b: np.sqrt(np.maximum(2 * L * (1 - np.sum(X[a] * X[b], -1)), 0))
    return d, nn, pair


def test_fp32_slack_with_spiky_variance():
    """Windows whose sigma differs by orders of magnitude inside one tile: the FP32 slack grows
    for the quiet windows (more cells reach the exact pass) and runs that walk out of a loud
    stretch restart from direct sums. The recurrence-based reference engine (and its C
    restatement) lose neighbours on this series; the drop-in must pick, for every offset, the
    nearest neighbour under the reference's own window statistics (prefix sums -- themselves
    ~1e-4 off for quiet windows after the loud stretch) with exact co-moments."""
    rng = np.random.default_rng(12)
    t = rng.standard_normal(6000) * 1e-3
    t[1000:1400] += rng.standard_normal(400) * 50.0
    t[4000:4600] += np.cumsum(rng.standard_normal(600)) * 20.0
    s = vl.ingest(t)
    run = api.GpuRun(s, 40, 48)
    assert run.stats["fp32_walk"] == 1
    for L in range(40, 49):
        mp, ip = run.profile(L)
        d, nn, pair = _brute_refstats(s, L)
        o = np.arange(ip.size)
        assert np.all(ip >= 0), L
        assert np.all(pair(o, ip) <= d * (1 + 1e-9)), L
        assert np.mean(ip == nn) > 0.999, L


def test_fp32_constant_stretches(oracle_mod):
    """Constant stretches put invalid windows (sigma below the floor: no neighbour, never a
    neighbour) inside tiles: their FP32 factors are +inf and the walk must neither pass nor
    poison their cells; valid offsets must still match the oracle exactly."""
    rng = np.random.default_rng(21)
    t = np.cumsum(rng.standard_normal(9000))
    # exact zeros: the prefix sums stay exactly flat, so sigma = 0 < floor (a constant stretch at
    # another level keeps prefix-sum noise above the floor: noise-decided in every implementation)
    t[2000:2600] = 0.0
    t[5000:5100] = 0.0
    s = vl.ingest(t)
    run = api.GpuRun(s, 50, 60)
    assert run.stats["fp32_walk"] == 1
    ref = oracle_mod.run(s, 50, 60, k_discord=1, keep_profiles=True)
    for L in range(50, 61):
        mp, ip = run.profile(L)
        omp, oip = ref["profiles"][L]
        assert np.array_equal(ip, oip), L
        fin = np.isfinite(omp)
        assert np.array_equal(fin, np.isfinite(mp)), L
        # reported values: the reference's pair_distance of the chosen pair (series.py:169-194);
        # the oracle's own STOMP-order values drift next to the flat stretches (ill-conditioned)
        cv = oracle_mod.canonical_values(s, ip, L)
        assert np.allclose(mp[fin], cv[fin], rtol=1e-12, atol=1e-12), L


def test_fp32_white_noise(oracle_mod):
    """White noise with short windows: weak correlations everywhere, the least favourable case
    for the bound filter (many passing cells, short runs). Profiles equal the oracle's."""
    t = np.random.default_rng(8).standard_normal(4000)
    s = vl.ingest(t)
    run = api.GpuRun(s, 10, 16)
    ref = oracle_mod.run(s, 10, 16, k_discord=1, keep_profiles=True)
    for L in range(10, 17):
        mp, ip = run.profile(L)
        omp, oip = ref["profiles"][L]
        assert np.array_equal(ip, oip), L
        assert np.allclose(mp, omp, rtol=1e-7, atol=1e-9)


def test_m_best_on_fp32_walk_spiky():
    """m-best mode (m-th discords) on the FP32 walk over the high dynamic-range series: each
    offset's m = 3 nearest neighbours equal the exact ones under the reference's statistics."""
    rng = np.random.default_rng(12)
    t = rng.standard_normal(6000) * 1e-3
    t[1000:1400] += rng.standard_normal(400) * 50.0
    t[4000:4600] += np.cumsum(rng.standard_normal(600)) * 20.0
    s = vl.ingest(t)
    sess = _lib.session(0)
    with sess.lock:
        sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
        sess.profile_mbest(40, 44, 3)
        got = {L: sess.profile_m_arrays(L) for L in range(40, 45)}
    for L in range(40, 45):
        d, nbr = got[L]
        W = np.lib.stride_tricks.sliding_window_view(t, L)
        mu = (s._cum[L:] - s._cum[:-L]) / L
        var = np.maximum((s._cum2[L:] - s._cum2[:-L]) / L - mu * mu, 0.0)
        X = (W - mu[:, None]) / np.sqrt(var * L)[:, None]
        N, e = W.shape[0], (L + 1) // 2
        idx = np.arange(N)
        for b0 in range(0, N, 1024):
            r2 = np.maximum(2 * L * (1 - X[b0:b0 + 1024] @ X.T), 0)
            r2[np.abs(idx[b0:b0 + 1024, None] - idx[None, :]) < e] = np.inf
            best = np.sort(r2, 1)[:, :3]
            mine = np.take_along_axis(r2, nbr[b0:b0 + 1024, :3], 1)
            assert np.allclose(np.sort(mine, 1), best, rtol=1e-9, atol=1e-12), (L, b0)
