"""The CPU oracle, pinned against fixtures produced by the REAL reference
(tests/golden/make_golden.py runs seriesmine here). CPU only."""

import numpy as np
import pytest

from conftest import SMALL_CASES, load_golden
from paper_2008_13447_b200 import ingest


def _motif_pairs(motifs):
    return [None if m is None else (m[0], m[1]) for m in motifs]


@pytest.mark.parametrize("name", SMALL_CASES)
def test_oracle_matches_reference_small(name, oracle_mod):
    g = load_golden(f"small_{name}")
    s = ingest(g["t"])
    lmin, lmax = int(g["lmin"]), int(g["lmax"])
    r = oracle_mod.run(s, lmin, lmax, k_discord=3, k_motif=1, ranking_capacity=10,
                       keep_profiles=True)
    # per-length profiles vs the reference's brute-force cdist oracle: IP exact
    for L in range(lmin, lmax + 1):
        mp, ip = r["profiles"][L]
        N = mp.shape[0]
        assert np.array_equal(ip, g["oracle_ip"][L - lmin, :N]), L
        fin = np.isfinite(g["oracle_mp"][L - lmin, :N])
        assert np.array_equal(fin, np.isfinite(mp))
        assert np.allclose(mp[fin], g["oracle_mp"][L - lmin, :N][fin], atol=1e-7)
    # VALMP vs the reference engine (valmod p=5) and its oracle
    assert np.array_equal(r["valmp_idx"], g["valmp_idx"])
    assert np.array_equal(r["valmp_len"], g["valmp_len"])
    assert np.array_equal(r["valmp_pop"], g["valmp_pop"])
    assert np.allclose(np.where(r["valmp_pop"], r["valmp_norm"], 0),
                       np.where(g["valmp_pop"], g["valmp_norm"], 0), atol=1e-7)
    # per-length top-1 motif (RunTrace.records[*].motif)
    want = [(int(a), int(b)) for a, b, _ in g["motif"]]
    assert _motif_pairs(r["motif"]) == want
    assert np.allclose([m[2] for m in r["motif"]], g["motif"][:, 2], atol=1e-7)
    # discords k=3, m=1, per length and merged
    assert np.array_equal(r["disc_off"], g["k3_disc_off"][:, :, 0])
    fin = np.isfinite(g["k3_disc_dist"][:, :, 0])
    assert np.allclose(r["disc_dist"][fin], g["k3_disc_dist"][:, :, 0][fin], atol=1e-7)
    assert np.array_equal(r["merged_off"], g["k3_merged_off"])
    assert np.array_equal(r["merged_len"], g["k3_merged_len"])
    # cross-length PairRanking(10)
    got = [(a, b, l) for a, b, l, _, _ in r["ranking"]]
    ref = [(int(x[0]), int(x[1]), int(x[2])) for x in g["ranking"]]
    assert got == ref


def test_oracle_degenerate_duplicates(oracle_mod):
    """Exact duplicate windows: d clamps to ~0 and the reference engine picks by
    rounding noise (its own brute-force oracle disagrees with it). The oracle must
    still report (near-)zero distances on genuinely duplicated pairs."""
    g = load_golden("small_dup11")
    s = ingest(g["t"])
    r = oracle_mod.run(s, int(g["lmin"]), int(g["lmax"]), keep_profiles=False)
    for m in r["motif"]:
        a, b, d = m
        assert d < 1e-5
        assert np.allclose(g["t"][a:a + 16], g["t"][b:b + 16])


def test_oracle_cfg1_against_reference(oracle_mod):
    g = load_golden("cfg1")
    s = ingest(g["t"])
    r = oracle_mod.run(s, 32, 64, k_discord=3, k_motif=3)
    assert np.array_equal(r["valmp_idx"], g["valmp_idx"])
    assert np.array_equal(r["valmp_len"], g["valmp_len"])
    assert np.allclose(r["valmp_norm"], g["valmp_norm"], atol=1e-7)
    want = [(int(a), int(b)) for a, b, _ in g["motif"]]
    assert _motif_pairs(r["motif"]) == want
    assert np.array_equal(r["disc_off"], g["k3_disc_off"][:, :, 0])
    assert np.array_equal(r["merged_off"], g["k3_merged_off"])
    for li, L in enumerate(range(32, 65)):
        ref = [(int(a), int(b)) for a, b, _ in g["top3_pairs"][li] if a >= 0]
        assert [(a, b) for a, b, _ in r["topk"][L]] == ref, L
    # survey anchors
    top = int(np.argmin(np.where(r["valmp_pop"], r["valmp_norm"], np.inf)))
    assert (top, int(r["valmp_idx"][top]), int(r["valmp_len"][top])) == (1661, 934, 62)
    assert r["motif"][0][:2] == (1080, 3853)
    assert int(r["disc_off"][0, 0]) == 3572


def test_oracle_kats(oracle_mod):
    """Known-answer tests from the reference suite (test_series.py:151-157,
    test_discords.py:20-35)."""
    s = ingest(np.array([1.0, 2.0, 3.0, 4.0, 4.0, 3.0, 2.0, 1.0, 5.0, 6.0]))
    # anti-correlated windows of length 4 -> distance 4.0
    assert oracle_mod.pair_distance(s, 0, 4, 4) == pytest.approx(4.0, abs=1e-12)
    # insertion policy: a weaker candidate below everything changes nothing
    d, o = oracle_mod.discords_m1(np.array([5.0, np.inf, 4.0, 3.0]), 4, 2)
    assert list(o) == [0, 2] and list(d) == [5.0, 4.0]   # offset 3 is trivial to 2


@pytest.mark.parametrize("seed", [10, 11, 12])
def test_oracle_m_th_discords_match_reference(seed, oracle_mod):
    """k = 3, m = 3 discords (discords.py:68-109) vs the reference engine's fixtures."""
    g = load_golden(f"small_m3_walk{seed}")
    s = ingest(g["t"])
    per, (md, mo, ml) = oracle_mod.discords_km(s, 16, 40, 3, 3)
    for L in range(16, 41):
        assert np.array_equal(per[L][1], g["k3m3_disc_off"][L - 16]), L
        fin = np.isfinite(g["k3m3_disc_dist"][L - 16])
        assert np.allclose(per[L][0][fin], g["k3m3_disc_dist"][L - 16][fin], atol=1e-7)
    assert np.array_equal(mo, g["k3m3_merged_off"]) and np.array_equal(ml, g["k3m3_merged_len"])


@pytest.mark.parametrize("name", ["cluster", "walk4"])
def test_motif_sets_oracle_rows_match_reference(name, oracle_mod):
    """The oracle's full-row range query + the package's admission pass (host code)
    reproduce the reference's compute_var_length_motif_sets on its own ranking."""
    from conftest import MOTIFSET_RF, golden_pairs, golden_sets
    from paper_2008_13447_b200.motifsets import expand_sets
    g = load_golden(f"motifsets_{name}")
    s = ingest(g["t"])
    pairs = golden_pairs(g)
    for tag, rf in MOTIFSET_RF.items():
        rows = []
        for p in pairs:
            r = p.distance * rf
            rows += [oracle_mod.range_row(s, p.off1, p.length, r),
                     oracle_mod.range_row(s, p.off2, p.length, r)]
        got = [(st.anchor, st.length, st.radius, st.members.tolist())
               for st in expand_sets(pairs, rows, rf)]
        assert got == golden_sets(g, tag), (name, tag)


def test_row_full_matches_reference_row_profile(oracle_mod):
    """oracle.row_full (direct dot products) against the reference's own row_profile
    (FFT correlation; tests/golden/make_rowprofile_golden.py): same +inf cells, distances and
    bound factors within 1e-9, dot products within 1e-9 relative."""
    g = load_golden("rowprofile")
    names = sorted({k[:-5] for k in g if k.endswith("_meta")})
    assert names
    for name in names:
        i, L = (int(x) for x in g[name + "_meta"])
        s = ingest(g[name.split("_")[0] + "_t"])
        d, f, qt = oracle_mod.row_full(s, i, L)
        rd, rf, rqt = g[name + "_dist"], g[name + "_f"], g[name + "_qt"]
        assert np.array_equal(np.isinf(d), np.isinf(rd)), name
        fin = np.isfinite(rd)
        assert np.allclose(d[fin], rd[fin], rtol=0, atol=1e-9), name
        assert np.allclose(f[fin], rf[fin], rtol=0, atol=1e-9), name
        assert np.allclose(qt, rqt, rtol=1e-9, atol=1e-9 * np.abs(rqt).max()), name
