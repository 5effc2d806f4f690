"""The pruned discord scan (MAD on the GPU, csrc/pruned.cu) through the C ABI:
it must return exactly the exhaustive path's matrices -- which are pinned to the reference's
own outputs (tests/golden) -- while recomputing only a fraction of the rows."""

import numpy as np
import pytest

import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import _lib, gen
from conftest import SMALL_CASES, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _device():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    _lib.load()


def _same(a, b):
    for L in a.per_length:
        assert np.array_equal(a.per_length[L].offset, b.per_length[L].offset), L
        assert np.array_equal(a.per_length[L].dist, b.per_length[L].dist), L
    assert np.array_equal(a.merged.offset, b.merged.offset)
    assert np.array_equal(a.merged.length, b.merged.length)
    assert np.array_equal(a.merged.dist, b.merged.dist)


@pytest.mark.parametrize("name", SMALL_CASES)
@pytest.mark.parametrize("k", [1, 3])
def test_pruned_matches_reference_small(name, k):
    g = load_golden(f"small_{name}")
    s = vl.ingest(g["t"])
    lmin, lmax = int(g["lmin"]), int(g["lmax"])
    trace = vl.RunTrace()
    scan = vl.topkm_discord_discovery(s, lmin, lmax, k, 1, 5, trace=trace, mode="pruned")
    for L in range(lmin, lmax + 1):
        assert np.array_equal(scan.per_length[L].offset, g[f"k{k}_disc_off"][L - lmin]), (name, L)
        fin = np.isfinite(g[f"k{k}_disc_dist"][L - lmin])
        assert np.allclose(scan.per_length[L].dist[fin], g[f"k{k}_disc_dist"][L - lmin][fin], atol=1e-7)
    assert np.array_equal(scan.merged.offset, g[f"k{k}_merged_off"])
    assert np.array_equal(scan.merged.length, g[f"k{k}_merged_len"])
    assert len(trace.records) == lmax - lmin + 1


@pytest.mark.parametrize("seed", [10, 11, 12])
def test_pruned_m_th_discords_match_reference(seed):
    """k = 3, m = 3 (stored entries P = min(8, p) = 5): the reference engine's matrices."""
    g = load_golden(f"small_m3_walk{seed}")
    s = vl.ingest(g["t"])
    scan = vl.topkm_discord_discovery(s, 16, 40, 3, 3, 5, mode="pruned")
    for L in range(16, 41):
        assert np.array_equal(scan.per_length[L].offset, g["k3m3_disc_off"][L - 16]), L
    assert np.array_equal(scan.merged.offset, g["k3m3_merged_off"])
    assert np.allclose(scan.merged.dist, g["k3m3_merged_dist"], atol=1e-7)


@pytest.mark.parametrize("seed,n,lmin,lmax,k,m,p", [
    (1, 5000, 40, 90, 3, 1, 8),
    (2, 8000, 64, 96, 5, 1, 4),
    (3, 6000, 50, 70, 4, 2, 8),
    (4, 3000, 24, 60, 8, 1, 1),     # P = 1: certification never holds, every candidate recomputed
])
def test_pruned_equals_exhaustive(seed, n, lmin, lmax, k, m, p):
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.standard_normal(n))
    t[n // 3:n // 3 + lmax] += rng.normal(0, 4.0, lmax)          # a planted discord
    s = vl.ingest(t)
    tr = vl.RunTrace()
    a = vl.topkm_discord_discovery(s, lmin, lmax, k, m, p, mode="exhaustive")
    b = vl.topkm_discord_discovery(s, lmin, lmax, k, m, p, trace=tr, mode="pruned")
    _same(a, b)
    rec = sum(r.n_recomputed for r in tr.records[1:])
    rows = sum(r.n_profiles for r in tr.records[1:])
    assert rec < rows            # pruning did something


def test_pruned_config1_matches_reference():
    g = load_golden("cfg1")
    s = vl.ingest(g["t"])
    for k in (1, 3):
        scan = vl.topkm_discord_discovery(s, 32, 64, k, 1, 50, mode="pruned")
        for L in range(32, 65):
            assert np.array_equal(scan.per_length[L].offset, g[f"k{k}_disc_off"][L - 32]), (k, L)
        assert np.array_equal(scan.merged.offset, g[f"k{k}_merged_off"])


def test_pruned_config2_matches_reference():
    """BASELINE config 2 at full size (129 lengths, k = 3) vs the reference engine's run."""
    g = load_golden("cfg2_discords")
    s = vl.ingest(gen.series_for(2))
    tr = vl.RunTrace()
    scan = vl.topkm_discord_discovery(s, 256, 384, 3, 1, 50, trace=tr, mode="pruned")
    for L in range(256, 385):
        assert np.array_equal(scan.per_length[L].offset, g["k3_disc_off"][L - 256]), L
        fin = np.isfinite(g["k3_disc_dist"][L - 256])
        assert np.allclose(scan.per_length[L].dist[fin], g["k3_disc_dist"][L - 256][fin], rtol=1e-6)
    assert np.array_equal(scan.merged.offset, g["k3_merged_off"])
    assert np.array_equal(scan.merged.length, g["k3_merged_len"])


@pytest.mark.slow
def test_pruned_config3_equals_exhaustive():
    """BASELINE config 3 (n = 262,144, quasi-periodic): 8 lengths, k = 5, both paths."""
    s = vl.ingest(gen.series_for(3))
    a = vl.topkm_discord_discovery(s, 480, 487, 5, 1, 50, mode="exhaustive")
    b = vl.topkm_discord_discovery(s, 480, 487, 5, 1, 50, mode="pruned")
    _same(a, b)
