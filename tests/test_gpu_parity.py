"""Parity of the CUDA path (through the C ABI) with the reference.

Anchors, in order of strength:
  * tests/golden/*.npz -- outputs of the REAL reference (seriesmine engine and its
    brute-force oracle), generated here by tests/golden/make_golden.py;
  * the CPU oracle (oracle/), itself pinned to those fixtures by
    test_oracle_golden.py, for cases without a fixture;
  * size-independent properties at BASELINE sizes (sampled row recomputes).
Tolerances: indices and lengths exact; distances 1e-7 absolute (the reference's
own tests, test_valmod.py:149-151) and <= 1e-6 relative (BASELINE north star).
"""

import numpy as np
import pytest

import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import _lib, api, gen
from conftest import SMALL_CASES, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _device():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    _lib.load()


def _gpu_run(t, lmin, lmax, flags=0):
    return api.GpuRun(vl.ingest(t), lmin, lmax, flags=flags)


@pytest.mark.parametrize("name", SMALL_CASES)
def test_valmod_matches_reference_small(name):
    g = load_golden(f"small_{name}")
    s = vl.ingest(g["t"])
    lmin, lmax = int(g["lmin"]), int(g["lmax"])
    trace = vl.RunTrace()
    ranking = vl.PairRanking(10)
    v = vl.valmod(s, lmin, lmax, 5, ranking=ranking, trace=trace)
    assert np.array_equal(v.indices, g["valmp_idx"])
    assert np.array_equal(v.lengths, g["valmp_len"])
    assert np.array_equal(v.populated, g["valmp_pop"])
    assert np.allclose(v.norm_distances[v.populated], g["valmp_norm"][g["valmp_pop"]], atol=1e-7)
    assert np.allclose(v.distances[v.populated], g["valmp_dist"][g["valmp_pop"]], atol=1e-7)
    got = [r.motif for r in trace.records]
    assert [m[:2] for m in got] == [(int(a), int(b)) for a, b, _ in g["motif"]]
    assert np.allclose([m[2] for m in got], g["motif"][:, 2], atol=1e-7)
    ref_rank = [(int(x[0]), int(x[1]), int(x[2])) for x in g["ranking"]]
    assert [(p.off1, p.off2, p.length) for p in ranking] == ref_rank
    assert np.allclose([p.norm_distance for p in ranking], g["ranking"][:, 4], atol=1e-7)
    top = vl.top_variable_length_motif(v)
    ref_top = int(np.argmin(np.where(g["valmp_pop"], g["valmp_norm"], np.inf)))
    assert top[0] == ref_top


@pytest.mark.parametrize("name", SMALL_CASES)
@pytest.mark.parametrize("k", [1, 3])
def test_discords_match_reference_small(name, k):
    g = load_golden(f"small_{name}")
    s = vl.ingest(g["t"])
    lmin, lmax = int(g["lmin"]), int(g["lmax"])
    trace = vl.RunTrace()
    scan = vl.topkm_discord_discovery(s, lmin, lmax, k, 1, 5, trace=trace)
    for L in range(lmin, lmax + 1):
        e, o = scan.per_length[L], g[f"k{k}_disc_off"][L - lmin]
        assert np.array_equal(e.offset, o), L
        fin = np.isfinite(g[f"k{k}_disc_dist"][L - lmin])
        assert np.allclose(e.dist[fin], g[f"k{k}_disc_dist"][L - lmin][fin], atol=1e-7)
    assert np.array_equal(scan.merged.offset, g[f"k{k}_merged_off"])
    assert np.array_equal(scan.merged.length, g[f"k{k}_merged_len"])
    assert np.allclose(scan.merged.dist, g[f"k{k}_merged_dist"], atol=1e-7)
    assert sum(r.n_recomputed for r in trace.records) == 0


@pytest.mark.parametrize("name", SMALL_CASES)
def test_profiles_match_reference_bruteforce(name):
    """Every per-length profile vs the reference's cdist oracle (IP exact)."""
    g = load_golden(f"small_{name}")
    lmin, lmax = int(g["lmin"]), int(g["lmax"])
    run = _gpu_run(g["t"], lmin, lmax)
    for L in range(lmin, lmax + 1):
        mp, ip = run.profile(L)
        N = mp.shape[0]
        assert np.array_equal(ip, g["oracle_ip"][L - lmin, :N]), L
        fin = np.isfinite(mp)
        assert np.array_equal(fin, np.isfinite(g["oracle_mp"][L - lmin, :N]))
        assert np.allclose(mp[fin], g["oracle_mp"][L - lmin, :N][fin], atol=1e-7)


@pytest.mark.parametrize("name", SMALL_CASES[:3])
def test_filter_mode_equals_full_fold_mode(name):
    """The bound-filtered kernel and the exact full-fold kernel pick identical neighbours."""
    g = load_golden(f"small_{name}")
    lmin, lmax = int(g["lmin"]), int(g["lmax"])
    a = _gpu_run(g["t"], lmin, lmax, flags=0)
    pa = [a.profile(L) for L in range(lmin, lmax + 1)]
    b = _gpu_run(g["t"], lmin, lmax, flags=_lib.FLAG_FULL_EVERY_LENGTH)
    for L, (mp, ip) in zip(range(lmin, lmax + 1), pa):
        mp2, ip2 = b.profile(L)
        assert np.array_equal(ip, ip2), L
        assert np.array_equal(mp, mp2), L


def test_cfg1_matches_reference():
    g = load_golden("cfg1")
    s = vl.ingest(g["t"])
    trace = vl.RunTrace()
    v = vl.valmod(s, 32, 64, 50, trace=trace)
    assert np.array_equal(v.indices, g["valmp_idx"])
    assert np.array_equal(v.lengths, g["valmp_len"])
    assert np.allclose(v.norm_distances, g["valmp_norm"], atol=1e-7)
    assert [r.motif[:2] for r in trace.records] == [(int(a), int(b)) for a, b, _ in g["motif"]]
    # SURVEY.md §8(c) anchor: pair {1661, 934} at length 62. The pair is mutual; with the
    # canonical symmetric distance both offsets tie exactly, as in the reference's own
    # brute-force oracle (first argmin -> 934); the reference engine's owner-first rows
    # differ by 1.4e-15 and report offset 1661 first.
    top = vl.top_variable_length_motif(v)
    assert {top[0], top[1]} == {934, 1661} and top[2] == 62
    assert top[4] == pytest.approx(0.1632923480786567, rel=1e-12)
    scan = vl.topkm_discord_discovery(s, 32, 64, 3, 1, 50)
    for L in range(32, 65):
        assert np.array_equal(scan.per_length[L].offset, g["k3_disc_off"][L - 32]), L
    assert np.array_equal(scan.merged.offset, g["k3_merged_off"])
    scan1 = vl.topkm_discord_discovery(s, 32, 64, 1, 1, 50)
    assert int(scan1.per_length[32].offset[0, 0]) == 3572   # SURVEY.md §8(c) anchor
    top3 = vl.motifs_per_length(s, 32, 64, 3)
    for L in range(32, 65):
        ref = [(int(a), int(b)) for a, b, _ in g["top3_pairs"][L - 32] if a >= 0]
        assert [(a, b) for a, b, _ in top3[L]] == ref, L
        refd = [d for a, _, d in g["top3_pairs"][L - 32] if a >= 0]
        assert np.allclose([d for _, _, d in top3[L]], refd, rtol=1e-6)


def test_cfg2_discords_match_reference():
    """Config 2 at full size (n=65,536, lengths 256..384, k=3) vs the reference engine."""
    g = load_golden("cfg2_discords")
    s = vl.ingest(gen.series_for(2))
    scan = vl.topkm_discord_discovery(s, 256, 384, 3, 1, 50)
    for L in range(256, 385):
        assert np.array_equal(scan.per_length[L].offset, g["k3_disc_off"][L - 256]), L
        fin = np.isfinite(g["k3_disc_dist"][L - 256])
        ref = g["k3_disc_dist"][L - 256][fin]
        assert np.allclose(scan.per_length[L].dist[fin], ref, rtol=1e-6)
    assert np.array_equal(scan.merged.offset, g["k3_merged_off"])
    assert np.array_equal(scan.merged.length, g["k3_merged_len"])


def test_cfg2_valmod_matches_reference():
    g = load_golden("cfg2_valmod")
    s = vl.ingest(gen.series_for(2))
    trace = vl.RunTrace()
    v = vl.valmod(s, 256, 384, 50, trace=trace)
    assert np.array_equal(v.lengths, g["valmp_len"])
    assert np.array_equal(v.indices, g["valmp_idx"])
    assert np.allclose(v.norm_distances, g["valmp_norm"], rtol=1e-6)
    assert [r.motif[:2] for r in trace.records] == [(int(a), int(b)) for a, b, _ in g["motif"]]


def test_cfg2_sampled_rows_against_oracle(oracle_mod):
    """Size-independent check at BASELINE config 2: random (row, length) profiles
    recomputed by the oracle's exhaustive row scan."""
    s = vl.ingest(gen.series_for(2))
    run = api.GpuRun(s, 256, 384)
    rng = np.random.default_rng(0)
    for L in (256, 300, 384):
        mp, ip = run.profile(L)
        rows = rng.integers(0, mp.shape[0], 24)
        for r in rows:
            omp, oip = oracle_mod.profile(s, L, nthreads=8, row_lo=int(r), row_hi=int(r) + 1)
            assert ip[r] == oip[r], (L, r)
            assert mp[r] == pytest.approx(omp[r], rel=1e-6, abs=1e-9)
    # the planted pair (5234, 10194) is the top motif around its length
    motifs = {r: None for r in range(1)}
    off, nbr, d = run.smallest_rows(1)
    assert sorted((int(off[300 - 256, 0]), int(nbr[300 - 256, 0]))) == [5234, 10194]


def test_cfg3_sampled_rows_against_oracle(oracle_mod):
    """Size-independent check at BASELINE config 3 (n = 262,144, lengths 400..600, a noisy
    sinusoid mixture with a planted discord): sampled (row, length) profiles recomputed by the
    oracle's exhaustive row scan, plus the planted discord among the top discords."""
    s = vl.ingest(gen.series_for(3))
    run = api.GpuRun(s, 400, 600)
    assert run.stats["fp32_walk"] == 1 and run.stats["exact_redo"] == 0
    rng = np.random.default_rng(3)
    for L in (400, 517, 600):
        mp, ip = run.profile(L)
        for r in rng.integers(0, mp.shape[0], 8):
            omp, oip = oracle_mod.profile(s, L, nthreads=8, row_lo=int(r), row_hi=int(r) + 1)
            if ip[r] != oip[r]:   # only an exact-arithmetic tie may pick another neighbour
                a = oracle_mod.pair_distance(s, r, ip[r], L); b = oracle_mod.pair_distance(s, r, oip[r], L)
                assert abs(a - b) <= 1e-9 * max(a, b), (L, r)
            assert mp[r] == pytest.approx(omp[r], rel=1e-6, abs=1e-9)
    _, d0 = gen.config3()
    dist, off = run.discords(1)
    o = int(off[500 - 400, 0])
    assert d0 - 500 < o < d0 + 500, (o, d0)   # the planted noise segment is the top discord


@pytest.mark.parametrize("case", ["constant_stretch", "dc_offset", "short", "spikes", "lmin4"])
def test_edge_cases_against_oracle(case, oracle_mod):
    rng = np.random.default_rng(7)
    lmin, lmax = 16, 40
    if case == "constant_stretch":
        t = np.cumsum(rng.standard_normal(900)); t[200:330] = 3.0; t[600:620] = -1.0
    elif case == "dc_offset":
        t = 1e4 + np.cumsum(rng.standard_normal(900))
    elif case == "short":
        t = np.cumsum(rng.standard_normal(lmax + (lmax + 1) // 2 + 1))
        lmin, lmax = 30, 40
    elif case == "spikes":
        t = np.sin(np.arange(1200) * 2 * np.pi / 50) + rng.normal(0, 0.05, 1200); t[300] += 6
    else:
        t = np.cumsum(rng.standard_normal(500)); lmin, lmax = 4, 12
    s = vl.ingest(t)
    ref = oracle_mod.run(s, lmin, lmax, k_discord=2, keep_profiles=True)
    run = api.GpuRun(s, lmin, lmax)
    for L in range(lmin, lmax + 1):
        mp, ip = run.profile(L)
        omp, oip = ref["profiles"][L]
        assert np.array_equal(ip, oip), (case, L)
        fin = np.isfinite(omp)
        assert np.array_equal(np.isfinite(mp), fin)
        # constant stretches create affine-copy windows (k constant samples + 1 step) whose
        # true distance is exactly 0; every evaluation returns rounding noise ~sqrt(eps*rho)
        # there (~3e-7; the oracle's own STOMP and pair formulas disagree by as much)
        atol = 1e-6 if case == "constant_stretch" else 1e-7
        assert np.allclose(mp[fin], omp[fin], rtol=1e-6, atol=atol)
    d, o = run.discords(2)
    assert np.array_equal(o, ref["disc_off"])
    v = run.valmp()
    robust = np.ones(v.indices.shape[0], dtype=bool)
    if case == "constant_stretch":
        # offsets whose best match is an exact affine copy (true distance 0): the winning
        # length is decided by ~1e-7 rounding noise in every implementation
        robust = ref["valmp_norm"] > 1e-5
    assert np.array_equal(v.indices[robust], ref["valmp_idx"][robust])
    assert np.array_equal(v.lengths[robust], ref["valmp_len"][robust])


def test_exact_duplicates_clamp_to_zero():
    """Duplicated windows: the radicand clamps to 0 and ties go to the smallest index
    (the reference engine resolves these by rounding noise; its brute-force oracle by
    exact zeros -- see DESIGN.md)."""
    g = load_golden("small_dup11")
    s = vl.ingest(g["t"])
    trace = vl.RunTrace()
    vl.valmod(s, 16, 32, 5, trace=trace)
    for rec in trace.records:
        a, b, d = rec.motif
        assert d < 1e-5
        assert np.allclose(g["t"][a:a + rec.length], g["t"][b:b + rec.length])


def test_compute_matrix_profile_and_errors(oracle_mod):
    s = vl.ingest(np.cumsum(np.random.default_rng(3).standard_normal(2000)))
    res = vl.compute_matrix_profile(s, 64, 5, m_track=1)
    omp, oip = oracle_mod.profile(s, 64)
    assert np.array_equal(res.profile.ip, oip)
    assert np.allclose(res.profile.mp, omp, atol=1e-7)
    assert np.array_equal(res.best_m_nbr[:, 0], oip)


def test_symmetric_values_for_mutual_pairs():
    """Canonical (min, max) evaluation: a mutual nearest-neighbour pair reports
    bitwise-equal distances from both owners (discords.py:126-141 requirement)."""
    s = vl.ingest(np.cumsum(np.random.default_rng(11).standard_normal(3000)))
    run = api.GpuRun(s, 40, 48)
    for L in (40, 44, 48):
        mp, ip = run.profile(L)
        mutual = np.flatnonzero((ip >= 0) & (ip[np.maximum(ip, 0)] == np.arange(ip.shape[0])))
        assert mutual.size > 10
        assert np.array_equal(mp[mutual], mp[ip[mutual]])


@pytest.mark.parametrize("seed", [10, 11, 12])
def test_m_th_discords_match_reference(seed):
    """Top-k m-th discords (k = 3, m = 3) vs the reference engine (discords.py:206-247)."""
    g = load_golden(f"small_m3_walk{seed}")
    s = vl.ingest(g["t"])
    scan = vl.topkm_discord_discovery(s, 16, 40, 3, 3, 5)
    for L in range(16, 41):
        assert np.array_equal(scan.per_length[L].offset, g["k3m3_disc_off"][L - 16]), L
        fin = np.isfinite(g["k3m3_disc_dist"][L - 16])
        assert np.allclose(scan.per_length[L].dist[fin], g["k3m3_disc_dist"][L - 16][fin], atol=1e-7)
    assert np.array_equal(scan.merged.offset, g["k3m3_merged_off"])
    assert np.array_equal(scan.merged.length, g["k3m3_merged_len"])
    assert np.allclose(scan.merged.dist, g["k3m3_merged_dist"], atol=1e-7)


@pytest.mark.parametrize("mb", [2, 4])
def test_m_best_rows_against_oracle(mb, oracle_mod):
    """compute_matrix_profile(m_track = m): the m best neighbours per row, exact, and their
    canonical distances ascending (profile.py:319-326, discords.py:126-141)."""
    s = vl.ingest(np.cumsum(np.random.default_rng(31).standard_normal(1500)))
    for L in (24, 40):
        res = vl.compute_matrix_profile(s, L, 5, m_track=mb)
        _, _, bm, bmi = oracle_mod.profile_m(s, L, mb)
        assert np.array_equal(np.sort(res.best_m_nbr, axis=1), np.sort(bmi, axis=1)), L
        fin = np.isfinite(bm)
        canon = np.sort(np.where(fin, bm, np.inf), axis=1)
        assert np.allclose(res.best_m[fin], canon[fin], atol=1e-7)


def test_m_th_discords_config1(oracle_mod):
    s = vl.ingest(gen.series_for(1))
    scan = vl.topkm_discord_discovery(s, 32, 40, 2, 3, 5)
    per, (md, mo, ml) = oracle_mod.discords_km(s, 32, 40, 2, 3)
    for L in range(32, 41):
        assert np.array_equal(scan.per_length[L].offset, per[L][1]), L
    assert np.array_equal(scan.merged.offset, mo)


def test_weak_bounds_fall_back_exactly(oracle_mod):
    """Short white noise: some offsets' best correlation is ~0 or negative, so their bound is
    too weak for the covariance-domain filter: those lengths run the
    exact full-fold body (1-best) and those offsets are recomputed exactly (m-best)."""
    s = vl.ingest(np.random.default_rng(5).standard_normal(61))
    lmin, lmax = 30, 40
    run = api.GpuRun(s, lmin, lmax)
    assert run.stats["fallback_lengths"] > 0
    ref = oracle_mod.run(s, lmin, lmax, k_discord=1, keep_profiles=True)
    for L in range(lmin, lmax + 1):
        mp, ip = run.profile(L)
        omp, oip = ref["profiles"][L]
        assert np.array_equal(ip, oip), L
        fin = np.isfinite(omp)
        assert np.allclose(mp[fin], omp[fin], rtol=1e-6, atol=1e-7)
    for L in (24, 30):
        res = vl.compute_matrix_profile(s, L, 5, m_track=3)
        _, _, bm, bmi = oracle_mod.profile_m(s, L, 3)
        assert np.array_equal(np.sort(res.best_m_nbr, axis=1), np.sort(bmi, axis=1)), L


@pytest.mark.parametrize("name", ["cluster", "walk4"])
def test_motif_sets_match_reference(name):
    """compute_var_length_motif_sets with GPU range queries, fed the reference's own
    ranking, reproduces the reference's sets (anchors, radius, members) exactly."""
    from conftest import MOTIFSET_RF, golden_pairs, golden_sets
    g = load_golden(f"motifsets_{name}")
    s = vl.ingest(g["t"])
    pairs = golden_pairs(g)
    for tag, rf in MOTIFSET_RF.items():
        sets = vl.compute_var_length_motif_sets(s, pairs, radius_factor=rf)
        got = [(st.anchor, st.length, st.radius, st.members.tolist()) for st in sets]
        assert got == golden_sets(g, tag), (name, tag)
        assert vl.validate_disjoint(sets)


def test_range_query_rows_against_oracle(oracle_mod):
    """vlmp_range_query rows equal the oracle's full-row range queries (several lengths,
    owners near both ends, radii around the row's own distance quantiles)."""
    from paper_2008_13447_b200.motifsets import range_members
    s = vl.ingest(np.cumsum(np.random.default_rng(41).standard_normal(3000)))
    rng = np.random.default_rng(3)
    owners, lengths, radii = [], [], []
    for L in (16, 57, 200):
        for o in (0, 1, 3000 - L, int(rng.integers(0, 3000 - L))):
            for rad in (1.0, 3.0, 6.0):
                owners.append(o); lengths.append(L); radii.append(rad * np.sqrt(L / 16.0))
    rows = range_members(s, owners, lengths, radii)
    for q in range(len(owners)):
        want = oracle_mod.range_row(s, owners[q], lengths[q], radii[q])
        assert np.array_equal(rows[q], want), (owners[q], lengths[q], radii[q])


def test_planted_cluster_motif_set_end_to_end():
    """GPU ranking (valmod) + GPU expansion on the reference's planted-cluster workload."""
    from conftest import golden_sets
    g = load_golden("motifsets_cluster")
    s = vl.ingest(g["t"])
    ranking = vl.PairRanking(10)
    vl.valmod(s, 32, 48, 8, ranking=ranking)
    sets = vl.compute_var_length_motif_sets(s, ranking, radius_factor=4.0)
    top = sorted(map(int, sets[0].members))
    assert sets[0].frequency == 5 and np.all(np.diff(top) == 300)   # the five planted copies
    ref_top = golden_sets(g, "rf4")[0]                               # the reference's own run
    assert (sets[0].anchor, sets[0].length, top) == (ref_top[0], ref_top[1], ref_top[3])


@pytest.mark.parametrize("scale", [1e-12, 1e-3, 1e6, 1e15])
def test_series_scale_invariance_against_oracle(scale, oracle_mod):
    """The filter's FP32 factors carry a per-series power-of-two scale (hi-word bias):
    profiles at extreme magnitudes still equal the oracle's exactly (indices) and use
    the filtered path (no full-fold fallback)."""
    t = scale * np.cumsum(np.random.default_rng(19).standard_normal(2500))
    s = vl.ingest(t)
    lmin, lmax = 24, 40
    run = api.GpuRun(s, lmin, lmax)
    assert run.stats["fallback_lengths"] == 0 and run.stats["exact_redo"] == 0
    ref = oracle_mod.run(s, lmin, lmax, k_discord=2, keep_profiles=True)
    for L in range(lmin, lmax + 1):
        mp, ip = run.profile(L)
        omp, oip = ref["profiles"][L]
        assert np.array_equal(ip, oip), (scale, L)
        fin = np.isfinite(omp)
        assert np.allclose(mp[fin], omp[fin], rtol=1e-7, atol=1e-9)
    d, o = run.discords(2)
    assert np.array_equal(o, ref["disc_off"])


def test_log_overflow_reruns_exactly(monkeypatch):
    """A candidate log too small for a length (forced with the VLMP_LOG_CAP test hook) drops
    candidates; the run is redone with full folds and the profiles equal the normal run."""
    s = vl.ingest(np.cumsum(np.random.default_rng(23).standard_normal(3000)))
    ref = api.GpuRun(s, 32, 48)
    want = [ref.profile(L) for L in range(32, 49)]
    assert ref.stats["exact_redo"] == 0
    monkeypatch.setenv("VLMP_LOG_CAP", "16")
    run = api.GpuRun(s, 32, 48)
    assert run.stats["exact_redo"] >= 1
    for L, (mp, ip) in zip(range(32, 49), want):
        got = run.profile(L)
        assert np.array_equal(got[1], ip) and np.array_equal(got[0], mp), L


def test_row_profile_matches_reference(oracle_mod):
    """row_profile (vlmp_row_profile, profile.py:263-269) against the reference's own
    row_profile fixtures (tests/golden/make_rowprofile_golden.py, FFT dot products) and against
    the oracle's direct-sum row on config 2's series."""
    g = load_golden("rowprofile")
    names = sorted({k[:-5] for k in g if k.endswith("_meta")})
    for name in names:
        i, L = (int(x) for x in g[name + "_meta"])
        s = vl.ingest(g[name.split("_")[0] + "_t"])
        d, f, qt = vl.row_profile(s, i, L, want_f=True)
        rd, rf, rqt = g[name + "_dist"], g[name + "_f"], g[name + "_qt"]
        assert np.array_equal(np.isinf(d), np.isinf(rd)), name
        fin = np.isfinite(rd)
        assert np.allclose(d[fin], rd[fin], rtol=0, atol=1e-9), name
        assert np.allclose(f[fin], rf[fin], rtol=0, atol=1e-9), name
        assert np.allclose(qt, rqt, rtol=1e-9, atol=1e-9 * np.abs(rqt).max()), name
        d2, f2, qt2 = vl.row_profile(s, i, L)
        assert f2 is None and np.array_equal(d2, d) and np.array_equal(qt2, qt)
    s = vl.ingest(gen.series_for(2))
    for i, L in ((0, 256), (5234, 300), (40000, 384), (s.n - 384, 384)):
        d, f, qt = vl.row_profile(s, i, L, want_f=True)
        od, of, oqt = oracle_mod.row_full(s, i, L)
        assert np.array_equal(np.isinf(d), np.isinf(od)), (i, L)
        fin = np.isfinite(od)
        assert np.allclose(d[fin], od[fin], rtol=1e-9, atol=1e-9), (i, L)
        assert np.allclose(f[fin], of[fin], rtol=1e-9, atol=1e-9), (i, L)
        j = int(np.argmin(d))     # the row's nearest neighbour equals the exhaustive profile's
        mp, ip = oracle_mod.profile(s, L, nthreads=1, row_lo=i, row_hi=i + 1)
        assert j == ip[i] or abs(d[j] - d[ip[i]]) <= 1e-9 * d[j], (i, L, j, ip[i])
    with pytest.raises(vl.OutOfRangeError):
        vl.row_profile(s, s.n - 10, 256)
    with pytest.raises(vl.SeriesTooShortError):
        vl.row_profile(s, 0, 3)


def test_mine_skips_read_offs_with_k_zero():
    """mine(k_motif=0) / mine(k_discord=0) (BASELINE configs 4 and 5 ask for only one of the
    two): the other read-offs equal a full mine() call's."""
    s = vl.ingest(np.cumsum(np.random.default_rng(3).standard_normal(3000)))
    full = vl.mine(s, 40, 50, k_motif=2, k_discord=2)
    no_d = vl.mine(s, 40, 50, k_motif=2, k_discord=0)
    no_m = vl.mine(s, 40, 50, k_motif=0, k_discord=2)
    assert no_d.motifs == full.motifs and no_m.motifs == {L: [] for L in range(40, 51)}
    assert np.array_equal(no_d.valmp.indices, full.valmp.indices)
    assert no_d.discords.merged.offset.shape == (0, 1)
    assert np.array_equal(no_m.discords.merged.offset, full.discords.merged.offset)
    for L in range(40, 51):
        assert np.array_equal(no_m.discords.per_length[L].offset, full.discords.per_length[L].offset)


@pytest.mark.parametrize("k2,k,want_v", [(6, 3, True), (2, 0, True), (0, 5, False), (4, 1, False)])
def test_finalize_collect_equals_separate_readoffs(k2, k, want_v):
    """vlmp_finalize_collect (phase 2 + read-offs, one host wait) returns exactly what
    vlmp_finalize + smallest_rows + discords + get_valmp return one by one."""
    s = vl.ingest(gen.series_for(1))
    sess = _lib.session(0)
    with sess.lock:
        sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
        sess.profile(32, 64, 0, -1, 0)
        sess.finalize()
        rows1 = sess.smallest_rows(k2) if k2 else None
        disc1 = sess.discords(k) if k else None
        v1 = sess.valmp_arrays()
        sess.profile(32, 64, 0, -1, 0)
        rows2, disc2, v2 = sess.finalize_collect(k2, k, want_v, end_event=1)
        v3 = sess.valmp_arrays()            # the session state after collect is finalized as usual
    if k2:
        assert all(np.array_equal(a, b) for a, b in zip(rows1, rows2))
    else:
        assert rows2 is None
    if k:
        assert all(np.array_equal(a, b) for a, b in zip(disc1, disc2))
    else:
        assert disc2 is None
    if want_v:
        assert all(np.array_equal(a, b) for a, b in zip(v1, v2))
    else:
        assert v2 is None
    assert all(np.array_equal(a, b) for a, b in zip(v1, v3))


def test_mine_collect_matches_separate_path():
    """mine() (collected read-offs) equals the same read-offs fetched one call at a time."""
    s = vl.ingest(gen.series_for(1))
    res = vl.mine(s, 32, 64, k_motif=3, k_discord=2)
    with api.GpuRun(s, 32, 64) as run:
        v = run.valmp()
        d, o = run.discords(2)
        motifs = api._topk_from_rows(run, 3)
    assert np.array_equal(res.valmp.indices, v.indices) and np.array_equal(res.valmp.distances, v.distances)
    assert res.motifs == motifs
    for li, L in enumerate(range(32, 65)):
        assert np.array_equal(res.discords.per_length[L].offset[:, 0], o[li])
