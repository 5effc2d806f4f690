"""Host-side logic of the drop-in (CPU only): argument validation with the
reference's error types, result-container semantics (reference KATs), ranking
threshold, generators, band partitioning."""

import numpy as np
import pytest

import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import api, gen, results
from paper_2008_13447_b200.exceptions import (AllConstantError, EmptySeriesError,
                                              InvalidParametersError, NonFiniteError,
                                              SeriesTooShortError, UnpopulatedError)


def walk(n, seed=0):
    return np.cumsum(np.random.default_rng(seed).standard_normal(n))


# --- validation happens before any device work (valmod.py:180-189, :213-214;
#     discords.py:214-218; profile.py:346-355) -----------------------------------
def test_valmod_range_validation():
    t = vl.ingest(walk(100, 9))
    with pytest.raises(InvalidParametersError):
        vl.valmod(t, 32, 16, 5)
    with pytest.raises(SeriesTooShortError):
        vl.valmod(t, 16, 80, 5)
    with pytest.raises(InvalidParametersError):
        vl.valmod(t, 8, 16, 0)
    with pytest.raises(InvalidParametersError):
        vl.valmod(t, 3, 16, 5)


def test_discord_parameter_validation():
    t = vl.ingest(walk(300, 23))
    with pytest.raises(InvalidParametersError) as exc:
        vl.topkm_discord_discovery(t, 16, 24, 1, 3, 2)
    assert "p" in str(exc.value) and "m" in str(exc.value)
    with pytest.raises(InvalidParametersError):
        vl.topkm_discord_discovery(t, 16, 24, 0, 1, 5)
    with pytest.raises(InvalidParametersError):   # m > 8 not on the GPU path (no CPU fallback)
        vl.topkm_discord_discovery(t, 16, 24, 1, 9, 9)


def test_all_constant_and_short():
    with pytest.raises(AllConstantError):
        vl.valmod(vl.ingest(np.ones(200)), 8, 16, 5)
    with pytest.raises(SeriesTooShortError):
        vl.compute_matrix_profile(vl.ingest(walk(20)), 12, 5)


def test_ingest_errors():
    with pytest.raises(EmptySeriesError):
        vl.ingest([])
    with pytest.raises(NonFiniteError) as exc:
        vl.ingest([1.0, np.nan, 2.0])
    assert exc.value.index == 1


def test_dataseries_matches_reference_prefix_sums():
    v = walk(1000, 3)
    s = vl.ingest(v)
    assert np.array_equal(s._cum[1:], np.cumsum(v))
    acc, out = 0.0, []
    for x in v:                      # np.cumsum is a sequential sum
        acc += x
        out.append(acc)
    assert np.array_equal(s._cum[1:], np.array(out))
    mu, sd = s.moving_stats(16)
    w = np.lib.stride_tricks.sliding_window_view(v, 16)
    assert np.allclose(mu, w.mean(1)) and np.allclose(sd, w.std(1))


# --- container semantics: reference KATs ----------------------------------------
def test_update_valmp_ties_keep_shorter_length():          # test_valmod.py:60-76
    v = vl.VALMP(4)
    mp = np.array([4.0, 2.0, 8.0, 1.0]); ip = np.array([2, 3, 0, 1])
    vl.update_valmp(v, mp, ip, 4, 16)
    assert v.populated.all() and np.allclose(v.norm_distances, mp / 4.0)
    vl.update_valmp(v, mp * np.sqrt(25 / 16), ip[::-1].copy(), 4, 25)
    assert np.all(v.lengths == 16) and np.array_equal(v.indices, ip)
    vl.update_valmp(v, mp * np.sqrt(25 / 16) * 0.5, ip[::-1].copy(), 4, 25)
    assert np.all(v.lengths == 25)


def test_top_motif_tie_and_unpopulated():                   # test_valmod.py:167-178
    v = vl.VALMP(5)
    vl.update_valmp(v, np.array([2.0, 1.0, 3.0, 1.0, 9.0]), np.array([3, 3, 0, 1, 0]), 5, 16)
    assert vl.top_variable_length_motif(v) == (1, 3, 16, 1.0, 0.25)
    with pytest.raises(UnpopulatedError):
        vl.top_variable_length_motif(vl.VALMP(4))


def test_ranking_semantics():                               # test_motifsets.py:21-38
    r = vl.PairRanking(8)
    assert r.push(10, 50, 1.0, 16, 0.25)
    assert not r.push(50, 10, 1.0, 16, 0.25)
    assert r.push(50, 10, 0.8, 16, 0.20)
    assert len(r) == 1 and next(iter(r)).norm_distance == 0.20
    r = vl.PairRanking(2)
    r.push(1, 20, 1.0, 8, 0.10); r.push(2, 30, 2.0, 8, 0.20)
    assert r.push(3, 40, 1.5, 8, 0.15)
    assert (2, 30) not in r and len(r) == 2


def test_discord_insertion_kats():                          # test_discords.py:20-35, :77-85
    dkm = vl.DiscordMatrix.empty(3, 2, 16)
    assert vl.update_fixed_length_discords(dkm, np.array([1.0, 2.0]), 50, 3, 2)
    assert dkm.dist[0, 1] == 2.0 and dkm.offset[0, 1] == 50
    merged = vl.VariableLengthDiscordMatrix.empty(1, 1)
    d16 = vl.DiscordMatrix.empty(1, 1, 16)
    vl.update_fixed_length_discords(d16, np.array([4.0]), 10, 1, 1)
    d25 = vl.DiscordMatrix.empty(1, 1, 25)
    vl.update_fixed_length_discords(d25, np.array([5.0]), 77, 1, 1)
    vl.update_variable_length_discords(d16, merged, 1, 1)
    vl.update_variable_length_discords(d25, merged, 1, 1)
    assert merged.length[0, 0] == 25 and merged.offset[0, 0] == 77


def test_ranking_threshold_bounds_every_final_pair():
    rng = np.random.default_rng(0)
    v = vl.VALMP(50)
    for length in (8, 9, 10):
        mp = rng.uniform(1, 5, 50)
        ip = (np.arange(50) + rng.integers(5, 40, 50)) % 50
        vl.update_valmp(v, mp, ip, 50, length)
    tau = api._ranking_threshold(v, 5)
    pairs = {}
    for i in np.flatnonzero(v.populated):
        a, b = sorted((int(i), int(v.indices[i])))
        key = (v.norm_distances[i], v.lengths[i], a, b)
        pairs[(a, b)] = min(pairs.get((a, b), key), key)
    kth = sorted(pairs.values())[4][0]
    assert tau == kth


def test_topk_from_rows_dedups_mirrored_pairs():
    class FakeRun:
        lmin = lmax = 16

        def smallest_rows(self, k2):
            off = np.array([[3, 9, 4, 1]]); nbr = np.array([[9, 3, 20, 30]])
            d = np.array([[1.0, 1.0, 2.0, 2.5]])
            return off, nbr, d
    out = api._topk_from_rows(FakeRun(), 2)
    assert out[16] == [(3, 9, 1.0), (4, 20, 2.0)]


# --- generators (SURVEY.md Appendix B anchors) ------------------------------------
def test_generators():
    assert np.array_equal(gen.config1(), np.cumsum(np.random.default_rng(0).standard_normal(4096)))
    t, (a, b) = gen.config2()
    assert (a, b) == (5234, 10194) and t.shape == (65536,)
    assert gen.pair_updates(4096, 32, 64) == 267350000 or abs(gen.pair_updates(4096, 32, 64) - 2.6735e8) < 1e5
    assert abs(gen.pair_updates(65536, 256, 384) / 2.7299e11 - 1) < 1e-4


def test_band_split_balances_work():
    from paper_2008_13447_b200 import distributed
    cuts = distributed.band_split(65536, 256, 384, 4)
    assert cuts[0] == 0 and cuts[-1] == distributed.n_bands(65536, 256)
    w = [sum(distributed.band_work(65536, 256, 384, b) for b in range(cuts[p], cuts[p + 1]))
         for p in range(4)]
    assert max(w) / min(w) < 1.05


def test_length_split_balances_and_covers():
    from paper_2008_13447_b200 import distributed as D
    for n, lmin, lmax in ((65536, 256, 384), (1 << 22, 1000, 1256), (6000, 48, 64)):
        nl = lmax - lmin + 1
        for parts in (1, 2, 3, 4, 8):
            c = D.length_split(n, lmin, lmax, parts)
            assert len(c) == parts + 1 and c[0] == 0 and c[-1] == nl and np.all(np.diff(c) >= 1)
            if nl >= 16 * parts:   # enough lengths per shard for the granularity to even out
                w = [sum(D.length_work(n, lmin + li) for li in range(c[p], c[p + 1])) for p in range(parts)]
                assert max(w) / min(w) < 1.1
    c = D.length_split(100, 10, 12, 8)          # more ranks than lengths: empty tail shards
    assert c.tolist() == [0, 1, 2, 3, 3, 3, 3, 3, 3]


@pytest.mark.parametrize("seed", range(6))
def test_batch_discord_merge_equals_sequential(seed):
    """mine()'s vectorised cross-length merge == update_variable_length_discords applied length
    by length (results.py; the reference's merge, discords.py), on ties across lengths, -inf
    (absent discords) and NaN cells."""
    from paper_2008_13447_b200.results import (DiscordMatrix, VariableLengthDiscordMatrix,
                                               merge_variable_length_discords,
                                               update_variable_length_discords)
    rng = np.random.default_rng(seed)
    nl, k, m = 9, 4, 2
    lengths = np.arange(30, 30 + nl)
    dist = rng.integers(0, 4, (nl, k, m)).astype(np.float64) * np.sqrt(lengths)[:, None, None]
    dist[rng.random((nl, k, m)) < 0.2] = -np.inf
    if seed % 2:
        dist[rng.random((nl, k, m)) < 0.15] = np.nan
    if seed == 5:
        dist[:, 0, 0] = np.nan
    off = rng.integers(-1, 500, (nl, k, m))
    seq = VariableLengthDiscordMatrix.empty(k, m)
    for li in range(nl):
        update_variable_length_discords(DiscordMatrix(dist[li].copy(), off[li].copy(), int(lengths[li])), seq, k, m)
    bat = merge_variable_length_discords(dist, off, lengths, VariableLengthDiscordMatrix.empty(k, m))
    assert np.array_equal(seq.dist, bat.dist)
    assert np.array_equal(seq.offset, bat.offset)
    assert np.array_equal(seq.length, bat.length)


def test_frontend_swaps_the_reference_entry_points():
    """paper_2008_13447_b200.frontend installs the drop-in into the reference's package and CLI
    (no GPU work: only the swap is checked); skipped when the reference is not installed."""
    import importlib
    import os
    import sys
    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "seriesmine")):
        pytest.skip("baseline/_ref not installed")
    from paper_2008_13447_b200 import frontend
    import paper_2008_13447_b200 as drop_in
    sm = frontend._import_reference()
    saved = {k: getattr(sm.cli, k) for k in ("valmod", "topkm_discord_discovery", "compute_matrix_profile",
                                            "compute_var_length_motif_sets")}
    saved_pkg = {k: getattr(sm, k) for k in ("valmod", "topkm_discord_discovery", "compute_var_length_motif_sets")}
    from paper_2008_13447_b200 import exceptions as dx
    saved_exc = {k: getattr(dx, k) for k in dx._NAMES}
    try:
        orig = frontend.swap_into(sm)
        assert orig["valmod"] is saved["valmod"]
        assert sm.cli.valmod is drop_in.valmod and sm.valmod is drop_in.valmod
        assert sm.cli.topkm_discord_discovery is drop_in.topkm_discord_discovery
        assert sm.cli.compute_matrix_profile is drop_in.compute_matrix_profile
        assert sm.cli.compute_var_length_motif_sets is drop_in.compute_var_length_motif_sets
        runner = frontend._gpu_bench_runner(sm, orig)
        assert callable(runner)
    finally:
        for k, v in saved.items():
            setattr(sm.cli, k, v)
        for k, v in saved_pkg.items():
            setattr(sm, k, v)
        for k, v in saved_exc.items():
            setattr(dx, k, v)
