"""The scalar Eq. 2 API (paper_2008_13447_b200/bounds.py) against its definition and the
reference's known answers (tests/test_bounds.py:47-56 of seriesmine: q = 0, L = 16 -> 4;
q = 1 -> 0), soundness on random extensions, scaling and O(1) entry updates."""

import numpy as np
import pytest

from paper_2008_13447_b200 import bounds as B
from paper_2008_13447_b200 import ingest
from paper_2008_13447_b200.exceptions import OutOfRangeError, ZeroVarianceError


def _zn(a, b):
    za = (a - a.mean()) / a.std()
    zb = (b - b.mean()) / b.std()
    return float(np.sqrt(((za - zb) ** 2).sum()))


def test_known_answers():
    assert B.lower_bound(0.0, 1.5, 1.5, 16).value == pytest.approx(4.0, rel=1e-12)
    assert B.lower_bound(1.0, 2.0, 3.0, 16).value == 0.0
    lb = B.lower_bound(-0.3, 2.0, 1.0, 9)            # q <= 0: sqrt(L) * ratio
    assert lb.value == pytest.approx(6.0) and (lb.base_length, lb.target_length) == (9, 10)
    with pytest.raises(ZeroVarianceError):
        B.lower_bound(0.5, 0.0, 1.0, 8)


def test_q_value_is_pearson_and_clamped():
    s = ingest(np.random.default_rng(1).standard_normal(300))
    for i, j in [(0, 64), (10, 150), (99, 40)]:
        a, b = s.window(i, 32), s.window(j, 32)
        q = B.q_value(float(a @ b), s.stats(i, 32), s.stats(j, 32))
        assert q == pytest.approx(float(np.corrcoef(a, b)[0, 1]), rel=1e-9)
    w = np.arange(1.0, 9.0)
    t = ingest(np.concatenate([w, w, -w]))
    assert B.q_value(float(w @ w), t.stats(0, 8), t.stats(8, 8)) == 1.0
    c = ingest(np.concatenate([np.full(8, 2.0), np.arange(8.0)]))
    with pytest.raises(ZeroVarianceError):
        B.q_value(16.0, c.stats(0, 8), c.stats(8, 8))


def test_bound_is_sound_on_random_extensions():
    rng = np.random.default_rng(2)
    s = ingest(np.cumsum(rng.standard_normal(500)))
    L = 32
    for _ in range(150):
        i, j = (int(x) for x in rng.integers(0, s.n - 2 * L, size=2))
        if abs(i - j) < L:
            continue
        q = B.q_value(float(s.window(i, L) @ s.window(j, L)), s.stats(i, L), s.stats(j, L))
        for k in range(1, L + 1):
            lb = B.lower_bound(q, s.stats(j, L).sigma, s.stats(j, L + k).sigma, L, L + k)
            assert lb.value <= _zn(s.window(i, L + k), s.window(j, L + k)) + 1e-9


def test_scale_bound_steps_equal_direct_and_keep_order():
    rng = np.random.default_rng(3)
    s = ingest(np.cumsum(rng.standard_normal(300)))
    L, i, j = 24, 10, 120
    q = B.q_value(float(s.window(i, L) @ s.window(j, L)), s.stats(i, L), s.stats(j, L))
    sg = lambda m: s.stats(j, m).sigma
    lb = B.lower_bound(q, sg(L), sg(L + 1), L)
    for m in (L + 1, L + 2):
        lb = B.scale_bound(lb, sg(m), sg(m + 1))
    direct = B.lower_bound(q, sg(L), sg(L + 3), L, L + 3)
    assert lb.value == pytest.approx(direct.value, rel=1e-12) and lb.target_length == L + 3
    many = [B.lower_bound(x, 1.0, 1.0, 16) for x in rng.uniform(-1, 1, 40)]
    before = np.argsort([b.value for b in many], kind="stable")
    after = np.argsort([B.scale_bound(b, 1.3, 0.7).value for b in many], kind="stable")
    assert np.array_equal(before, after)


def test_update_dist_and_lb_tracks_scratch_and_ends():
    rng = np.random.default_rng(6)
    s = ingest(np.cumsum(rng.standard_normal(1000)))
    i, j, L = 40, 500, 16
    e = B.ProfileEntry(i, j, float(s.window(i, L) @ s.window(j, L)), 0.0, 0.0)
    for m in range(17, 33):
        e = B.update_dist_and_lb(e, s, m)
        assert e.dist == pytest.approx(_zn(s.window(i, m), s.window(j, m)), abs=1e-7)
        assert 0.0 <= e.lb
    short = ingest(np.cumsum(rng.standard_normal(40)))
    e = B.ProfileEntry(20, 0, float(short.window(20, 19) @ short.window(0, 19)), 0.0, 0.0)
    e = B.update_dist_and_lb(e, short, 20)        # the owner's window now ends the series
    assert np.isnan(e.lb) and np.isfinite(e.dist)
    with pytest.raises(OutOfRangeError):
        B.update_dist_and_lb(e, short, 21)
